"""K1 rasterization-group sweep: time (CUDA events, prequeued) at the config-2 K1 shapes.

    KVPR_GEMM_GROUP_M=<g> python tools/k1_group_probe.py   (unset = the library's L2-band default)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_17089_b200 import kernels  # noqa: E402

dev = torch.device("cuda:0")
b, h = 32, 4096
w = (torch.randn(2 * h, h, device=dev) * 0.02).half()
bias = (torch.randn(2 * h, device=dev) * 0.02).half()
pages = torch.empty(1056, 2, b, h, dtype=torch.float16, device=dev)
for l in (296, 592, 895):
    x = torch.randn(l, b, h, device=dev).half()
    for _ in range(3):
        kernels.recompute_kv(x, w, bias, pages, b, 0, l)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(1e8))
    s.record()
    for _ in range(10):
        kernels.recompute_kv(x, w, bias, pages, b, 0, l)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 10 / 1e3
    print(json.dumps({"group_m": os.environ.get("KVPR_GEMM_GROUP_M", "default"), "l": l, "M": b * l,
                      "us": round(t * 1e6, 1), "tflops": round(4 * b * l * h * h / t / 1e12, 1)}), flush=True)
