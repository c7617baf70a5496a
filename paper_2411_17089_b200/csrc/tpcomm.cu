// Fused TP projection + all-reduce over peer memory (BASELINE config 4: OPT-30B head-sharded over
// the GPUs of one NVSwitch domain).
//
// A row-parallel projection (out-proj, fc2) ends in an all-reduce of the fp32 residual.  Instead of
// GEMM -> NCCL all-reduce, every rank runs two kernels back to back (PDL-chained):
//
//   1. push   the swap-AB decode GEMM (csrc/gemm_tcgen05.cu, tp_world > 1): each 128-column tile's
//             raw fp32 partial is stored straight into slot [rank] of the tile OWNER's receive buffer
//             (owner = tile % world) over NVLink, then the owner's flag (rank, tile) is released at
//             system scope.  The partials leave the SM while the other tiles are still in the MMA.
//   2. reduce every rank sums the slots of the tiles it owns in rank order (deterministic), adds
//             the bias and its residual, stores the result into EVERY rank's residual (NVLink
//             stores) and releases their broadcast flags; the kernel ends only when the broadcast
//             flags of all tiles have arrived in this rank, so the next kernel reads a complete
//             residual.
//
// Reduce-scatter + all-gather of 1 x the fp32 partial per rank, with no host involvement and no
// staging copies.  Flags carry a per-call epoch (wrap-safe compare), so nothing is ever reset.
// Peer buffers are CUDA IPC allocations (kvpr_ipc_*) exchanged by the host (tp.PeerBuffers).
//
// Ordering (why no buffer is overwritten while a peer still reads it): a rank's push for call k+1
// follows its own reduce kernel of call k, which finished only after every tile of call k was
// broadcast, i.e. after every owner finished reading its slots for call k.  The owner's broadcast
// into rank d's residual for call k needs d's push of call k, which follows (stream order) every
// kernel of d that read the residual before the projection.

#include <string.h>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {

namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *f has reached `epoch` (wrap-safe).  A peer that never arrives sets *err and lets the
// kernel finish (garbage out, loud error on the host) instead of hanging the GPU.
__device__ bool wait_flag(const unsigned* f, unsigned epoch, unsigned* err) {
  const unsigned long long t0 = globaltimer();
  while (static_cast<int>(ld_acquire_sys(f) - epoch) < 0) {
    __nanosleep(128);
    if (globaltimer() - t0 > 5000000000ull) {
      atomicExch(err, 1u);
      return false;
    }
  }
  return true;
}

struct TpReduceArgs {
  int M, N, T, rank, world;
  unsigned epoch;
  const __half* bias;
  const float* recv;                // this rank's slots [world][M][N]
  unsigned* flags;                  // this rank's flags: [world][kTpMaxTiles] push, [kTpMaxTiles] bcast
  float* resid[kTpMaxWorld];        // every rank's residual [M][N]
  unsigned* peer_flags[kTpMaxWorld];
  unsigned* err;
};

constexpr int kReduceThreads = 256;
constexpr int kTileCols = 128;

__global__ void __launch_bounds__(kReduceThreads) tp_reduce_kernel(const TpReduceArgs a) {
  pdl_trigger();
  pdl_wait();
  const int W = a.world;
  for (int t = a.rank + W * blockIdx.x; t < a.T; t += W * gridDim.x) {
    if (threadIdx.x < W) wait_flag(a.flags + threadIdx.x * kTpMaxTiles + t, a.epoch, a.err);
    __syncthreads();
    const int n0 = t * kTileCols;
    for (int idx = threadIdx.x; idx < a.M * kTileCols; idx += kReduceThreads) {
      const int m = idx / kTileCols, n = n0 + idx % kTileCols;
      if (n >= a.N) continue;
      const long long off = static_cast<long long>(m) * a.N + n;
      float v = 0.f;
      for (int r = 0; r < W; ++r) v += a.recv[static_cast<long long>(r) * a.M * a.N + off];  // rank order
      if (a.bias != nullptr) v += __half2float(a.bias[n]);
      const float out = a.resid[a.rank][off] + v;
      for (int d = 0; d < W; ++d) a.resid[d][off] = out;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < W) st_release_sys(a.peer_flags[threadIdx.x] + W * kTpMaxTiles + t, a.epoch);
    __syncthreads();
  }
  // the whole residual (every owner's broadcast) has landed here before this kernel completes
  for (int t = blockIdx.x * kReduceThreads + threadIdx.x; t < a.T; t += gridDim.x * kReduceThreads)
    wait_flag(a.flags + W * kTpMaxTiles + t, a.epoch, a.err);
}

}  // namespace

}  // namespace kvpr

using namespace kvpr;

extern "C" {

size_t kvpr_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int kvpr_ipc_alloc(size_t bytes, void** dptr, void* handle) {
  clear_error();
  if (bytes == 0 || dptr == nullptr || handle == nullptr) {
    set_error("ipc_alloc: zero size or null output");
    return KVPR_EINVAL;
  }
  cudaError_t e = cudaMalloc(dptr, bytes);
  if (e == cudaSuccess) e = cudaMemset(*dptr, 0, bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), *dptr);
  if (e != cudaSuccess) {
    set_error("ipc_alloc: %s", cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}

int kvpr_ipc_open(const void* handle, void** dptr) {
  clear_error();
  if (handle == nullptr || dptr == nullptr) {
    set_error("ipc_open: null handle or output");
    return KVPR_EINVAL;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error("ipc_open: %s", cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}

int kvpr_ipc_close(void* dptr) {
  return cudaIpcCloseMemHandle(dptr) == cudaSuccess ? KVPR_OK : KVPR_ECUDA;
}

int kvpr_ipc_free(void* dptr) { return cudaFree(dptr) == cudaSuccess ? KVPR_OK : KVPR_ECUDA; }

int kvpr_linear_allreduce(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                          const void* bias, const kvpr_tp_peers* peers, unsigned epoch, void* stream) {
  clear_error();
  if (a == nullptr || w == nullptr || peers == nullptr || peers->world < 2 || peers->world > kTpMaxWorld ||
      peers->rank < 0 || peers->rank >= peers->world || peers->err == nullptr) {
    set_error("linear_allreduce: bad arguments (world must be 2..%d)", kTpMaxWorld);
    return KVPR_EINVAL;
  }
  for (int r = 0; r < peers->world; ++r) {
    if (peers->recv[r] == nullptr || peers->resid[r] == nullptr || peers->flags[r] == nullptr) {
      set_error("linear_allreduce: peer %d buffers missing", r);
      return KVPR_EINVAL;
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GemmArgs tp;
  memset(&tp, 0, sizeof(tp));
  tp.tp_rank = peers->rank;
  tp.tp_world = peers->world;
  tp.tp_epoch = epoch;
  tp.scale = 1.f;
  for (int r = 0; r < peers->world; ++r) {
    tp.tp_recv[r] = static_cast<float*>(peers->recv[r]);
    tp.tp_flags[r] = peers->flags[r];
  }
  int rc = gemm_tp_partials(a, lda, w, ldw, M, N, K, tp, s);
  if (rc) return rc;
  TpReduceArgs ra;
  memset(&ra, 0, sizeof(ra));
  ra.M = M;
  ra.N = N;
  ra.T = (N + kTileCols - 1) / kTileCols;
  ra.rank = peers->rank;
  ra.world = peers->world;
  ra.epoch = epoch;
  ra.bias = static_cast<const __half*>(bias);
  ra.recv = static_cast<const float*>(peers->recv[peers->rank]);
  ra.flags = peers->flags[peers->rank];
  for (int r = 0; r < peers->world; ++r) {
    ra.resid[r] = peers->resid[r];
    ra.peer_flags[r] = peers->flags[r];
  }
  ra.err = peers->err;
  const int owned = (ra.T + ra.world - 1) / ra.world;
  return launch("tp_reduce", tp_reduce_kernel, owned, kReduceThreads, 0, s, ra);
}

}  // extern "C"
