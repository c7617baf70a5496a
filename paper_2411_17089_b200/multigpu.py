"""Multi-GPU host logic for the batch-partitioned mode (BASELINE config 3).

Sequences are independent units: the global batch is split
into contiguous slices, one per rank (one process per GPU, launched by
torchrun), and every rank runs its own KVPRRuntime with its own page-locked
host stores, its own PCIe link, its own live profile and its own plan (l
depends on b only through the transfer latency, scheduler.py:113-115).
There is no collective on the data path; the only cross-rank traffic is the
timing reduction (max over ranks) and the final token gather on the host.
The paper's multi-GPU experiment is the same shape: independent processes,
no collectives.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .costmodel import ModelSpec, WorkloadSpec
from .hwprofile import HardwareProfile
from .scheduler import SplitPlan, plan_generation


@dataclass(frozen=True)
class Slice:
    rank: int
    start: int
    count: int


def partition(global_batch: int, world: int) -> list[Slice]:
    """Contiguous slices whose sizes differ by at most one (first ranks take the remainder)."""
    if global_batch < world or world <= 0:
        raise ValueError(f"cannot split batch {global_batch} over {world} ranks")
    base, rem = divmod(global_batch, world)
    out, p = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append(Slice(r, p, n))
        p += n
    return out


def rank_workload(wl: WorkloadSpec, sl: Slice) -> WorkloadSpec:
    return WorkloadSpec(batch_size=sl.count, prompt_len=wl.prompt_len, gen_len=wl.gen_len,
                        num_batches=wl.num_batches, kv_bytes_per_element=wl.kv_bytes_per_element)


def rank_plan(spec: ModelSpec, wl: WorkloadSpec, profile: HardwareProfile, world: int, rank: int,
              mode: str = "column") -> SplitPlan:
    """The plan rank `rank` executes: the reference solver on its own slice and its own profile."""
    return plan_generation(spec, rank_workload(wl, partition(wl.batch_size, world)[rank]), profile, mode)


def max_over_ranks(value: float, device: torch.device | None = None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_tokens(local: torch.Tensor, global_batch: int, device: torch.device | None = None) -> torch.Tensor:
    """[steps, b_local] per rank -> [steps, global_batch] on every rank, sequences in global order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    slices = partition(global_batch, world)
    width = max(s.count for s in slices)
    steps = local.shape[0]
    dev = device or local.device
    pad = torch.full((steps, width), -1, dtype=torch.int64, device=dev)
    pad[:, : local.shape[1]] = local.to(dev, torch.int64)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([bufs[s.rank][:, : s.count] for s in slices], dim=1)


# ---------------------------------------------------------------------------
# NUMA placement of a rank's host stores
#
# Every rank streams X[:, :l] and KV[l:] from its own page-locked stores over its own PCIe link;
# on a two-socket host those pages must sit on the socket the GPU's root port hangs off, or every
# H2D crosses the inter-socket link (and all ranks share it).  Pinning faults pages in on the
# calling thread, so restricting the rank to the GPU's local CPUs before the stores are allocated
# places them locally (first touch).

def parse_cpulist(text: str) -> list[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11] (the kernel's cpulist format)."""
    out: list[int] = []
    for part in text.strip().split(","):
        part = part.strip()
        if not part:
            continue
        if "-" in part:
            lo, hi = part.split("-", 1)
            if int(hi) < int(lo):
                raise ValueError(f"bad cpulist range {part!r}")
            out.extend(range(int(lo), int(hi) + 1))
        else:
            out.append(int(part))
    return sorted(set(out))


def pci_address(device_index: int) -> str:
    p = torch.cuda.get_device_properties(device_index)
    return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"


def bind_to_gpu_numa(device_index: int, sysfs: str = "/sys/bus/pci/devices") -> dict:
    """Restrict this process to the CPUs local to GPU `device_index` (no-op on one-node hosts).

    Returns what was done: {"pci", "numa_node", "cpus", "bound"}.
    """
    import os
    from pathlib import Path

    info: dict = {"pci": None, "numa_node": None, "cpus": None, "bound": False}
    try:
        addr = pci_address(device_index)
        info["pci"] = addr
        d = Path(sysfs) / addr
        node = int((d / "numa_node").read_text().strip()) if (d / "numa_node").exists() else -1
        info["numa_node"] = node
        cpus = parse_cpulist((d / "local_cpulist").read_text()) if (d / "local_cpulist").exists() else []
        allowed = sorted(os.sched_getaffinity(0))
        local = [c for c in cpus if c in set(allowed)]
        info["cpus"] = len(local)
        if local and len(local) < len(allowed):
            os.sched_setaffinity(0, local)
            info["bound"] = True
    except (OSError, ValueError, RuntimeError, AttributeError) as e:
        info["error"] = str(e)
    return info
