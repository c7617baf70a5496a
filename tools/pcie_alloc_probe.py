"""Pinned-host allocation flavours vs H2D / D2H copy-engine bandwidth (1 GiB copies, CUDA events):
cudaHostRegister of pageable memory (the runtime's host stores), cudaHostAlloc default (torch
pin_memory), cudaHostAlloc write-combined.

    python tools/pcie_alloc_probe.py > gpurun_out/pcie_alloc.jsonl
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt is None:
    for cand in ("libcudart.so", "libcudart.so.12"):
        try:
            rt = ctypes.CDLL(cand)
            break
        except OSError:
            pass
N = 1 << 30
dev = torch.empty(N, dtype=torch.uint8, device="cuda")


def bw(host_ptr, direction, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    cudaMemcpyAsync = rt.cudaMemcpyAsync
    cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(reps):
        s.record()
        if direction == "h2d":
            cudaMemcpyAsync(dev.data_ptr(), host_ptr, N, 1, st)
        else:
            cudaMemcpyAsync(host_ptr, dev.data_ptr(), N, 2, st)
        e.record()
        e.synchronize()
        best = max(best, N / (s.elapsed_time(e) / 1e3) / 1e9)
    return best


out = {}
# 1. cudaHostRegister of pageable memory
t = torch.empty(N, dtype=torch.uint8)
t.fill_(1)
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
assert rt.cudaHostRegister(ctypes.c_void_p(t.data_ptr()), N, 0) == 0
out["registered"] = {"h2d": bw(t.data_ptr(), "h2d"), "d2h": bw(t.data_ptr(), "d2h")}
rt.cudaHostUnregister(ctypes.c_void_p(t.data_ptr()))
# 2/3. cudaHostAlloc default / write-combined
for name, flags in (("hostalloc", 0), ("hostalloc_wc", 4)):
    p = ctypes.c_void_p()
    rt.cudaHostAlloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
    assert rt.cudaHostAlloc(ctypes.byref(p), N, flags) == 0
    ctypes.memset(p, 1, N)
    out[name] = {"h2d": bw(p.value, "h2d"), "d2h": bw(p.value, "d2h")}
    rt.cudaFreeHost(p)
print(json.dumps(out))
