"""B200-native KVPR decode path (arXiv 2411.17089): KV cache offloaded to host DRAM,
per layer X[:, :l] shipped over PCIe and K,V[0:l] recomputed on the GPU (tcgen05 GEMM)
while KV[l:s'] streams concurrently, split l from the reference's cost model.

Modules mirroring the reference package ``kvoverlap`` (same names and errors):
    costmodel, hwprofile, scheduler, numerics (GPU), cli
B200 runtime and tooling:
    profiler (live PCIe / GEMM probes), runtime (streams, events, pinned stores),
    tp (head-sharded tensor parallelism), multigpu (batch partition), trace
    (measured timelines in the reference's schema), weights (OPT geometry + init),
    kernels / _lib (ctypes binding of libkvpr.so, include/kvpr.h)
"""

__version__ = "0.1.0"
