"""Is one DMA stream enough to saturate H2D?  1 GiB pinned -> HBM as 1, 2 or 4 concurrent copies."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2411_17089_b200 import _lib

n = 1 << 30
host = torch.empty(n, dtype=torch.uint8)
host.fill_(1)
torch.cuda.cudart().cudaHostRegister(host.data_ptr(), n, 0)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
res = {}
for k in (1, 2, 4):
    for rep in range(4):
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s0.record(torch.cuda.current_stream())
        ends = []
        for i in range(k):
            st = streams[i]
            st.wait_event(s0)
            part = n // k
            _lib.call("kvpr_copy_async", dev.data_ptr() + i * part, host.data_ptr() + i * part, part, st.cuda_stream)
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            ends.append(e)
        torch.cuda.synchronize()
        t = max(s0.elapsed_time(e) for e in ends) / 1e3
        res.setdefault(k, []).append(n / t / 1e9)
print(json.dumps({f"{k}_streams_gbs": max(v) for k, v in res.items()}))
# H2D while a D2H runs (full duplex)
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
host2 = torch.empty(n, dtype=torch.uint8)
torch.cuda.cudart().cudaHostRegister(host2.data_ptr(), n, 0)
torch.cuda.synchronize()
s0 = torch.cuda.Event(enable_timing=True)
s0.record(torch.cuda.current_stream())
streams[0].wait_event(s0)
streams[1].wait_event(s0)
_lib.call("kvpr_copy_async", dev.data_ptr(), host.data_ptr(), n, streams[0].cuda_stream)
_lib.call("kvpr_copy_async", host2.data_ptr(), d2.data_ptr(), n, streams[1].cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(streams[0])
e1.record(streams[1])
torch.cuda.synchronize()
print(json.dumps({"duplex_h2d_gbs": n / (s0.elapsed_time(e0) / 1e3) / 1e9,
                  "duplex_d2h_gbs": n / (s0.elapsed_time(e1) / 1e3) / 1e9}))
