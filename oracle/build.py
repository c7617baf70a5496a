"""Build the oracle's C helpers (TEST INFRASTRUCTURE ONLY): oracle/libfp16conv.so.

    python -m oracle.build          # or via __graft_entry__.build()

gcc only; the .so is git-ignored but travels to the GPU box with the snapshot.  Without it
opt_ref falls back to NumPy's (slower, bit-identical) float16 casts."""

from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB = HERE / "libfp16conv.so"


def build(force: bool = False) -> Path | None:
    src = HERE / "csrc" / "fp16conv.c"
    if not force and LIB.exists() and LIB.stat().st_mtime >= src.stat().st_mtime:
        return LIB
    gcc = shutil.which("gcc")
    if gcc is None:
        return None
    subprocess.run([gcc, "-O3", "-mavx2", "-mf16c", "-fopenmp", "-shared", "-fPIC", str(src), "-o", str(LIB), "-lm"],
                   check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
