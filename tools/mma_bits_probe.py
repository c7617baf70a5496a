"""Does the warp-level mma.sync m16n8k16 (fp16 in, fp32 accumulate, k ascending in 16-wide steps)
reproduce the bits of the tcgen05 kernels (same k order)?  Compares kvpr_debug_mma_linear with the
swap-AB decode GEMM (kvpr_linear, bn -1, fp32 out, no bias) on random operands.

    python tools/mma_bits_probe.py > gpurun_out/mma_bits.json
"""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2411_17089_b200 import _lib, kernels  # noqa: E402

lib = _lib.load()
lib.kvpr_debug_mma_linear.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
out = []
for (M, N, K, scale) in [(4, 2304, 768, 1.0), (4, 1536, 768, 0.05), (8, 1024, 1024, 1.0), (1, 512, 4096, 1.0),
                         (4, 2304, 768, 30.0)]:
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    a = (torch.randn(M, K, generator=g) * scale).half().cuda()
    w = (torch.randn(N, K, generator=g) * 0.05).half().cuda()
    o1 = torch.empty(M, N, dtype=torch.float32, device="cuda")
    o2 = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    kernels.linear_simple(a, w, None, o1, bn=-1)
    rc = lib.kvpr_debug_mma_linear(a.data_ptr(), w.data_ptr(), o2.data_ptr(), M, N, K, None)
    torch.cuda.synchronize()
    ref = a.double() @ w.double().T
    diff = (o1 != o2).sum().item()
    out.append({"M": M, "N": N, "K": K, "rc": rc, "mismatches": diff, "of": M * N,
                "max_abs_diff": (o1 - o2).abs().max().item(),
                "tcgen05_err": (o1.double() - ref).abs().max().item(), "mma_err": (o2.double() - ref).abs().max().item()})
print(json.dumps(out))
