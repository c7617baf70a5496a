"""Live profiler: the B200 measures its own PCIe and recompute rates.

KVPR's profiler -> scheduler -> runtime chain.  The
reference replaces the profiler with hand-entered CSV records fed to
``calibrate`` (hwprofile.py:108-166); here the records are produced on the
device with CUDA events:

  h2d / d2h : pinned host (the host stores' allocation, hostmem.py) <-> HBM copies of 2^24..2^30
              bytes on a dedicated copy stream (the runtime's transfer path,
              kvpr_copy_async);
  gemm      : the K1 recompute GEMM itself (kvpr_recompute_kv) at several
              prefix lengths of the target model, size = 4*b*l*h^2 FLOPs
              (costmodel.recompute_flops).

The records go through the unchanged least-squares fit (hwprofile.calibrate),
and the resulting HardwareProfile feeds the bit-exact split solver.
"""

from __future__ import annotations

import statistics

import torch

from . import _lib, kernels
from .hostmem import pinned_empty, unpin
from .hwprofile import CalibrationResult, Measurement, calibrate


def _time(fn, stream: torch.cuda.Stream, reps: int, warm: int = 2) -> float:
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts)


def probe_transfers(device=None, sizes=(1 << 24, 1 << 26, 1 << 28, 1 << 30), reps: int = 5) -> list[Measurement]:
    dev = torch.device(device or "cuda")
    big = max(sizes)
    host = pinned_empty((big,), torch.uint8)  # the host stores' allocation (hostmem)
    host.fill_(1)
    try:
        d = torch.empty(big, dtype=torch.uint8, device=dev)
        s = torch.cuda.Stream(dev)
        out = []
        for n in sizes:
            h2d = lambda: _lib.call("kvpr_copy_async", d.data_ptr(), host.data_ptr(), n, s.cuda_stream)  # noqa: E731
            d2h = lambda: _lib.call("kvpr_copy_async", host.data_ptr(), d.data_ptr(), n, s.cuda_stream)  # noqa: E731
            out.append(Measurement("h2d", float(n), _time(h2d, s, reps)))
            out.append(Measurement("d2h", float(n), _time(d2h, s, reps)))
        del d
        return out
    finally:
        unpin(host)


def probe_recompute(hidden: int, batch: int, prefix_lens=(128, 256, 512, 1024), device=None,
                    reps: int = 5) -> list[Measurement]:
    dev = torch.device(device or "cuda")
    lmax = max(prefix_lens)
    g = torch.Generator(device=dev)
    g.manual_seed(123)
    x = torch.randn(lmax, batch, hidden, device=dev, generator=g).half()
    w = (torch.randn(2 * hidden, hidden, device=dev, generator=g) * 0.02).half()
    bias = torch.zeros(2 * hidden, device=dev, dtype=torch.float16)
    pages = torch.empty(lmax, 2, batch, hidden, device=dev, dtype=torch.float16)
    s = torch.cuda.Stream(dev)
    out = []
    for l in prefix_lens:
        fn = lambda: kernels.recompute_kv(x, w, bias, pages, batch, 0, l, stream=s)  # noqa: E731
        out.append(Measurement("gemm", float(4 * batch * l * hidden * hidden), _time(fn, s, reps)))
    return out


def measure(hidden: int, batch: int, device=None, sizes=(1 << 24, 1 << 26, 1 << 28, 1 << 30),
            prefix_lens=(128, 256, 512, 1024)) -> tuple[CalibrationResult, list[Measurement]]:
    """Probe this GPU and fit a HardwareProfile with the reference's calibration."""
    recs = probe_transfers(device, sizes) + probe_recompute(hidden, batch, prefix_lens, device)
    return calibrate(recs), recs


def peak_h2d(records: list[Measurement]) -> float:
    """Best pinned H2D bytes/s among the records (the roofline's BW_h2d)."""
    return max(m.size / m.elapsed_s for m in records if m.kind == "h2d")
