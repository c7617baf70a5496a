"""Per-SM streaming bandwidth with plain 16-byte loads/stores (kvpr_debug_sm_pull on device memory):
GB/s of a 1 GiB device-to-device copy driven by 1..148 CTAs (one per SM).  Compares with the ~46 GB/s
per SM the TMA-fed decode GEMMs reach."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_17089_b200 import _lib  # noqa: E402

N = 1 << 30
src = torch.empty(N, dtype=torch.uint8, device="cuda")
dst = torch.empty(N, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
res = {}
for ctas in (1, 2, 4, 8, 16, 32, 74, 148, 296):
    n = N if ctas >= 16 else N // 8
    _lib.call("kvpr_debug_sm_pull", src.data_ptr(), dst.data_ptr(), n, ctas, s.cuda_stream)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.call("kvpr_debug_sm_pull", src.data_ptr(), dst.data_ptr(), n, ctas, s.cuda_stream)
    e.record()
    e.synchronize()
    t = a.elapsed_time(e) / 1e3
    res[ctas] = {"read_gbs": round(n / t / 1e9, 1), "read_gbs_per_cta": round(n / t / 1e9 / ctas, 1)}
print(json.dumps(res))
