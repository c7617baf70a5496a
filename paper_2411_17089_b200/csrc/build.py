"""Build libkvpr.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2411_17089_b200.csrc.build      # or via __graft_entry__.build()

The shared library is written next to the package (paper_2411_17089_b200/libkvpr.so)
so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parent
PKG = CSRC.parent
ROOT = PKG.parent
LIB = PKG / "libkvpr.so"
SOURCES = ["abi.cu", "gemm_tcgen05.cu", "attention.cu", "elementwise.cu", "kvquant.cu", "executor.cu", "tpcomm.cu", "gemv.cu", "layer_tail.cu", "prefill_attn.cu", "sched_engine.cu"]
HEADERS = ["common.cuh", "kvpr_internal.h", "attn_common.cuh"]

NVCC_FLAGS = [
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if os.path.exists(cand) else "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "kvpr.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    objs = []
    tmp = CSRC / "_obj"
    tmp.mkdir(exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = tmp / (Path(src).stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        if os.environ.get("KVPR_GEMM_TRACE") == "1":  # tools/sk_trace.py: per-CTA timestamps in the decode GEMM
            cmd.insert(1, "-DKVPR_GEMM_TRACE")
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(str(obj))
    failed = False
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or (verbose and out):
            sys.stderr.write(" ".join(cmd) + "\n" + out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed building libkvpr.so")
    link = [nvc for nvc in [nvcc()]] + ["-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", str(LIB)]
    subprocess.run(link, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
