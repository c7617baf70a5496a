"""Why is K2 slower inside the decode step than standalone?  Time it (CUDA events) in
three situations at the config-2 shape: back-to-back, after the GPU idled ~5 ms (as between
PCIe-bound layers), and right after a 75 MB H2D into the same page buffer."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2411_17089_b200 import _lib, kernels

dev = torch.device("cuda")
b, h, s = 32, 4096, 1025
pages = torch.randn(1056, 2, b, h, device=dev).half()
q = torch.randn(b, h, device=dev).half()
out = torch.empty(b, h, device=dev).half()
ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
host = torch.empty(75 << 20, dtype=torch.uint8)
torch.cuda.cudart().cudaHostRegister(host.data_ptr(), host.numel(), 0)
cs = torch.cuda.current_stream()


def timed(fn):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    e.record()
    e.synchronize()
    return a.elapsed_time(e) * 1e3


k2 = lambda: kernels.decode_attention(q, pages, out, ws, b, 32, 128, s)  # noqa: E731
for _ in range(5):
    k2()
res = {"back_to_back_us": sorted(timed(k2) for _ in range(10))[5]}
idle = []
for _ in range(10):
    torch.cuda.synchronize()
    time.sleep(0.005)
    idle.append(timed(k2))
res["after_5ms_idle_us"] = sorted(idle)[5]
after = []
for _ in range(10):
    _lib.call("kvpr_copy_async", pages[900].data_ptr(), host.data_ptr(), host.numel(), cs.cuda_stream)
    after.append(timed(k2))
res["after_h2d_us"] = sorted(after)[5]
spin = []
for _ in range(10):  # GPU kept busy (a long GEMM) right before K2
    x = torch.randn(4096, 4096, device=dev).half()
    torch.cuda.synchronize()
    y = x @ x
    spin.append(timed(k2))
res["after_busy_gemm_us"] = sorted(spin)[5]
res["bytes"] = 2 * b * s * h * 2
print(json.dumps(res))

# K2 while a copy engine streams into / out of HBM on another stream (as the next layer's
# X chunks and KV tail do in the step).
big = torch.empty(1 << 30, dtype=torch.uint8)
torch.cuda.cudart().cudaHostRegister(big.data_ptr(), big.numel(), 0)
dst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
side = torch.cuda.Stream()
for name, d2h in (("concurrent_h2d_us", False), ("concurrent_d2h_us", True)):
    conc = []
    for _ in range(10):
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            if d2h:
                big.copy_(dst, non_blocking=True)
            else:
                dst.copy_(big, non_blocking=True)
        time.sleep(0.002)
        conc.append(timed(k2))
    torch.cuda.synchronize()
    res[name] = sorted(conc)[5]
print(json.dumps(res))

# Is the slowdown K2's access pattern or any HBM-streaming kernel?  A 512 MiB device-to-device
# copy by SM threads (torch copy kernel), alone and with the same concurrent H2D.
src2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
dst2 = torch.empty_like(src2)
smcopy = lambda: dst2.copy_(src2)  # noqa: E731
for _ in range(3):
    smcopy()
res["sm_copy_alone_us"] = sorted(timed(smcopy) for _ in range(10))[5]
conc = []
for _ in range(10):
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        dst.copy_(big, non_blocking=True)
    time.sleep(0.002)
    conc.append(timed(smcopy))
torch.cuda.synchronize()
res["sm_copy_concurrent_h2d_us"] = sorted(conc)[5]
res["sm_copy_bytes"] = 2 * src2.numel()
print(json.dumps(res))
