"""Per-CTA timing of the stream-K decode GEMM (globaltimer stamps, kvpr_debug_gemm_trace).

    KVPR_GEMM_TRACE=1 python -m paper_2411_17089_b200.csrc.build --force   # stamps compiled in
    python tools/sk_trace.py [M N K] > gpurun_out/sk_trace.json
stamps per CTA (ns from the earliest start): 0 start, 1..3 epilogue got segment 1..3's accumulator,
4 fixup reduce begins (last arriver), 5 exit."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2411_17089_b200 import _lib, kernels

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 4096, 4096)
dev = torch.device("cuda")
lib = _lib.load()
lib.kvpr_debug_gemm_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(148 * 8, dtype=torch.int64, device=dev)
ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
mats = [(torch.randn(N, K, device=dev) * 0.02).half() for _ in range(max(2, (320 << 20) // (N * K * 2)))]
a = (torch.randn(M, K, device=dev) * 0.5).half()
o = torch.empty(M, N, device=dev)
for i in range(5):
    kernels.linear_simple(a, mats[i % len(mats)], None, o, bn=-1, ws=ws)
torch.cuda.synchronize()
lib.kvpr_debug_gemm_trace(ctypes.c_void_p(buf.data_ptr()))
kernels.linear_simple(a, mats[-1], None, o, bn=-1, ws=ws)
torch.cuda.synchronize()
lib.kvpr_debug_gemm_trace(None)
t = buf.view(148, 8).cpu().tolist()
t0 = min(r[0] for r in t if r[0])
rows = [[(x - t0) if x else None for x in r[:8]] for r in t]
print(json.dumps({"M": M, "N": N, "K": K, "ctas": rows}))
ends = sorted(r[5] for r in rows if r[5] is not None)
starts = sorted(r[0] for r in rows if r[0] is not None)
seg = sorted(max(x for x in r[1:4] if x is not None) for r in rows if r[1] is not None)
fix = sorted(r[4] for r in rows if r[4] is not None)
print(json.dumps({"start_ns": [starts[0], starts[-1]], "last_acc_ns": [seg[0], seg[len(seg) // 2], seg[-1]],
                  "fixup_begin_ns": [fix[0], fix[-1]] if fix else None, "exit_ns": [ends[0], ends[len(ends) // 2], ends[-1]]}),
      file=sys.stderr)
d = sorted((r[5] - max(x for x in r[1:4] if x is not None), i) for i, r in enumerate(rows) if r[5] is not None and r[1] is not None)
print(json.dumps({"last_acc_to_exit_ns": [d[0], d[len(d) // 2], d[-1]]}), file=sys.stderr)
red = [r for r in rows if r[4] is not None]
print(json.dumps({"reducers": [[r[4], r[6], r[7], r[5]] for r in sorted(red, key=lambda r: -r[5])[:6]]}), file=sys.stderr)
