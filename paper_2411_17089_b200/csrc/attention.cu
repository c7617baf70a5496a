// K2: split-KV decode attention over the merged (recomputed + transferred)
// KV pages, read in place (the causal prefill attention is prefill_attn.cu).
//
// Reference semantics: numerics.decode_attention (numerics.py:166-191) —
// per head, softmax(K q / sqrt(d)) V with the max-subtracted softmax of
// numerics.py:159-163; the merged cache of numerics.split_merge_kv
// (numerics.py:134-137) is never materialised: positions [0,l) were written
// by K1, [l,s'-1) by the H2D copy, s'-1 by the decode-token projection, all
// into the same page buffer.
//
// Memory pattern: a page holds K (then V) of one position for all sequences,
// so one (sequence, head) row of K is 2*head_dim contiguous bytes.  A group of
// head_dim/8 lanes owns one position and each lane moves 16 B (128-bit
// loads), so every request is whole 32-byte sectors.  Scores reduce with
// xor-shuffles inside the lane group; the online softmax state (m, l, acc)
// is merged across groups and warps at the end, and across splits by the
// combine kernel (log-sum-exp merge).

#include <math.h>

#include <stdlib.h>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kvpr_internal.h"
#include "attn_common.cuh"

namespace kvpr {

namespace cg = cooperative_groups;
using namespace attn;

namespace {

constexpr int kMaxClusterSplits = 8;  // portable cluster size

// grid: (batch*heads, splits), block: 128 threads.  Q4: positions [q4.lo, q4.hi) come from
// compressed pages (the caller passes base/page_bytes/lo/hi; per-lane offsets are set here).
// CL: the splits of one (sequence, head) form a thread-block cluster; every split writes its
// softmax state into the cluster leader's shared memory (DSMEM) and the leader merges them in
// split order -- the same arithmetic as decode_attn_combine_kernel, without the second launch
// or the round trip through global memory.
template <int D, bool Q4, bool CL>
__global__ void __launch_bounds__(128) decode_attn_kernel(const __half* __restrict__ q, const __half* __restrict__ kv,
                                                          __half* __restrict__ out, float* __restrict__ ws, int batch,
                                                          int heads, int seq_len, int chunk, float qscale, Q4Src q4,
                                                          const int* __restrict__ seq_lens) {
  constexpr int LPP = D / 8;
  constexpr int PPW = 32 / LPP;  // positions per warp step
  constexpr int NW = 4;
  pdl_trigger();
  // DSMEM rule: a CTA may touch a peer's shared memory only once every CTA of the cluster has
  // started; the arrival here and the wait just before the remote stores cost nothing in between
  if constexpr (CL) {
    if (gridDim.y > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  }
  pdl_wait();  // q (qkv GEMM), pages [0, l) (K1) come from the preceding kernels
  const int bh = blockIdx.x;
  const int b = bh / heads;
  const int hd = bh % heads;
  const int hidden = heads * D;
  const int split = blockIdx.y;
  // ragged batches (seq_lens != nullptr): sequence b attends over its own [0, seq_lens[b]) of the
  // padded slab; a split past its end contributes an empty state (m = -inf), dropped by the merge
  const int len_b = seq_lens != nullptr ? min(seq_len, __ldg(seq_lens + b)) : seq_len;
  const int p_lo = split * chunk;
  const int p_hi = min(len_b, p_lo + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int glane = lane % LPP, grp = lane / LPP;

  float q8[8];
  load8(q + (long long)b * hidden + hd * D + glane * 8, q8);
#pragma unroll
  for (int i = 0; i < 8; ++i) q8[i] *= qscale;

  const long long page_stride = 2LL * batch * hidden;
  const __half* kbase = kv + (long long)b * hidden + hd * D;
  Softmax8 st;
  st.init();
  if constexpr (Q4) {
    const long long e = (long long)b * hidden + hd * D + glane * 8;  // element index of this lane's K slice
    q4.ck = e / 2;
    q4.cv = q4.ck + (long long)batch * hidden / 2;
    q4.pk = (long long)batch * hidden + (e / 64) * 4;  // params follow the 2*batch*hidden/2 code bytes
    q4.pv = q4.pk + ((long long)batch * hidden / 64) * 4;
  }
  sweep<D, 4, Q4>(kbase, page_stride, (long long)batch * hidden, p_lo + warp * PPW, p_hi, NW * PPW, grp, q8, glane, st,
                  &q4);
  merge_in_warp<LPP>(st);

  __shared__ float sm_m[NW], sm_l[NW];
  __shared__ float sm_acc[NW][D];
  __shared__ float sm_part[CL ? kMaxClusterSplits : 1][D + 2];  // cluster leader: every split's state
  if (lane < LPP) {
    if (lane == 0) {
      sm_m[warp] = st.m;
      sm_l[warp] = st.l;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) sm_acc[warp][glane * 8 + i] = st.acc[i];
  }
  __syncthreads();
  if constexpr (CL) {
    if (gridDim.y > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }
  if (threadIdx.x < D) {
    const int dd = threadIdx.x;
    float m = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) m = fmaxf(m, sm_m[w]);
    float l = 0.f, a = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float f = (sm_m[w] == -INFINITY) ? 0.f : exp2f(sm_m[w] - m);
      l += sm_l[w] * f;
      a += sm_acc[w][dd] * f;
    }
    if (gridDim.y == 1) {
      out[(long long)b * hidden + hd * D + dd] = __float2half_rn(a / l);
    } else if constexpr (CL) {
      float* w = cg::this_cluster().map_shared_rank(&sm_part[0][0], 0) + split * (D + 2);
      w[2 + dd] = a;
      if (dd == 0) {
        w[0] = m;
        w[1] = l;
      }
    } else {
      float* w = ws + ((long long)bh * gridDim.y + split) * (D + 2);
      w[2 + dd] = a;
      if (dd == 0) {
        w[0] = m;
        w[1] = l;
      }
    }
  }
  if constexpr (CL) {
    if (gridDim.y > 1) {
      cg::this_cluster().sync();  // every split's state is in the leader's smem
      if (split == 0 && threadIdx.x < D) {
        const int dd = threadIdx.x;
        const int splits = gridDim.y;
        float m = -INFINITY;
        for (int s2 = 0; s2 < splits; ++s2) m = fmaxf(m, sm_part[s2][0]);
        float l = 0.f, a = 0.f;
        for (int s2 = 0; s2 < splits; ++s2) {
          const float ms = sm_part[s2][0];
          const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - m);
          l += sm_part[s2][1] * f;
          a += sm_part[s2][2 + dd] * f;
        }
        out[(long long)b * hidden + hd * D + dd] = __float2half_rn(a / l);
      }
    }
  }
}

// grid: batch*heads, block: D threads — log-sum-exp merge of the split partials.
template <int D>
__global__ void decode_attn_combine_kernel(const float* __restrict__ ws, __half* __restrict__ out, int heads,
                                           int splits) {
  pdl_trigger();
  pdl_wait();
  const int bh = blockIdx.x;
  const int b = bh / heads, hd = bh % heads;
  const int dd = threadIdx.x;
  const float* w = ws + (long long)bh * splits * (D + 2);
  float m = -INFINITY;
  for (int s = 0; s < splits; ++s) m = fmaxf(m, w[s * (D + 2)]);
  float l = 0.f, a = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float ms = w[s * (D + 2)];
    const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - m);
    l += w[s * (D + 2) + 1] * f;
    a += w[s * (D + 2) + 2 + dd] * f;
  }
  out[(long long)b * heads * D + hd * D + dd] = __float2half_rn(a / l);
}

// (bh, splits) grid in clusters of (1, splits): one cluster per (sequence, head), PDL-chained
template <typename... KArgs, typename... Args>
int launch_cluster(void (*kern)(KArgs...), dim3 grid, int splits, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = splits;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    set_error("decode_attention (cluster): launch failed: %s", cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return check_launch("decode_attention");
}

}  // namespace

int decode_attention(const __half* q, const __half* kv, __half* out, float* ws, size_t ws_bytes, int batch, int heads,
                     int head_dim, int seq_len, float scale, cudaStream_t stream, const int* seq_lens) {
  return decode_attention_q4(q, kv, nullptr, 0, 0, out, ws, ws_bytes, batch, heads, head_dim, seq_len, scale, stream,
                             seq_lens);
}

int decode_attention_q4(const __half* q, const __half* kv, const uint8_t* qpages, int q_lo, int q_hi, __half* out,
                        float* ws, size_t ws_bytes, int batch, int heads, int head_dim, int seq_len, float scale,
                        cudaStream_t stream, const int* seq_lens) {
  const bool use_q4 = q_hi > q_lo;
  if (use_q4 && (qpages == nullptr || q_lo < 0 || q_hi > seq_len || (heads * head_dim) % 64 != 0 ||
                 (reinterpret_cast<uintptr_t>(qpages) & 3))) {
    set_error("decode_attention_kv4: need 4-byte aligned qpages, 0 <= q_lo <= q_hi <= seq_len, hidden %% 64 == 0 "
              "(got [%d,%d) of %d)", q_lo, q_hi, seq_len);
    return KVPR_EINVAL;
  }
  if (seq_len <= 0) {
    set_error("cannot attend over an empty cache (seq_len=%d)", seq_len);
    return KVPR_EINVAL;
  }
  if (batch <= 0 || heads <= 0 || (head_dim != 64 && head_dim != 128)) {
    set_error("decode_attention: batch=%d heads=%d head_dim=%d (head_dim must be 64 or 128)", batch, heads, head_dim);
    return KVPR_EINVAL;
  }
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv)) & 15) {
    set_error("decode_attention: q / kv must be 16-byte aligned");
    return KVPR_EINVAL;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  const int bh = batch * heads;
  // CTAs per SM the split-KV grid aims for (each split >= 64 positions); KVPR_K2_CTAS_PER_SM
  // overrides for experiments
  static int per_sm = -1;
  if (per_sm < 0) {
    const char* e = getenv("KVPR_K2_CTAS_PER_SM");
    per_sm = (e != nullptr && atoi(e) > 0) ? atoi(e) : 8;
  }
  const int target = per_sm * sm_count(dev);
  int splits = (target + bh - 1) / bh;
  static int min_pos = -1;  // positions per split at least (KVPR_K2_MIN_POS overrides for experiments)
  if (min_pos < 0) {
    const char* e = getenv("KVPR_K2_MIN_POS");
    min_pos = (e != nullptr && atoi(e) > 0) ? atoi(e) : 64;
  }
  const int max_by_len = (seq_len + min_pos - 1) / min_pos;
  if (splits > max_by_len) splits = max_by_len;
  // up to kMaxClusterSplits splits merge in the cluster leader's smem (no workspace); more need the
  // fp32 partials in ws and the combine kernel
  const size_t per_split = (size_t)bh * (head_dim + 2) * sizeof(float);
  if (splits > kMaxClusterSplits) {
    if (ws == nullptr || ws_bytes < per_split) splits = kMaxClusterSplits;
    else if ((size_t)splits * per_split > ws_bytes) splits = (int)(ws_bytes / per_split);
    if (splits < kMaxClusterSplits) splits = kMaxClusterSplits;
  }
  if (splits < 1) splits = 1;
  const int chunk = (seq_len + splits - 1) / splits;
  splits = (seq_len + chunk - 1) / chunk;
  const float qscale = scale * kLog2e;
  dim3 grid(bh, splits);
  Q4Src q4{};
  if (use_q4) {
    q4.base = qpages;
    q4.page_bytes = (long long)kv4_page_bytes(batch, heads * head_dim);
    q4.lo = q_lo;
    q4.hi = q_hi;
  }
  // KVPR_K2_CLUSTER=0: merge with the combine kernel instead (A/B tests; read per call so a test can
  // flip it, a getenv is ~100 ns against a >= 5 us kernel)
  const char* cl_env = getenv("KVPR_K2_CLUSTER");
  const bool cluster_merge = !(cl_env != nullptr && cl_env[0] == '0') || ws == nullptr;
  if (splits > 1 && splits <= kMaxClusterSplits && cluster_merge) {  // merge in DSMEM: one launch
    if (head_dim == 128)
      return use_q4 ? launch_cluster(decode_attn_kernel<128, true, true>, grid, splits, stream, q, kv, out, ws, batch,
                                     heads, seq_len, chunk, qscale, q4, seq_lens)
                    : launch_cluster(decode_attn_kernel<128, false, true>, grid, splits, stream, q, kv, out, ws, batch,
                                     heads, seq_len, chunk, qscale, q4, seq_lens);
    return use_q4 ? launch_cluster(decode_attn_kernel<64, true, true>, grid, splits, stream, q, kv, out, ws, batch,
                                   heads, seq_len, chunk, qscale, q4, seq_lens)
                  : launch_cluster(decode_attn_kernel<64, false, true>, grid, splits, stream, q, kv, out, ws, batch,
                                   heads, seq_len, chunk, qscale, q4, seq_lens);
  }
  int rc;
  if (head_dim == 128) {
    if (use_q4)
      rc = launch("decode_attention", decode_attn_kernel<128, true, false>, grid, 128, 0, stream, q, kv, out, ws,
                  batch, heads, seq_len, chunk, qscale, q4, seq_lens);
    else
      rc = launch("decode_attention", decode_attn_kernel<128, false, false>, grid, 128, 0, stream, q, kv, out, ws,
                  batch, heads, seq_len, chunk, qscale, q4, seq_lens);
  } else {
    if (use_q4)
      rc = launch("decode_attention", decode_attn_kernel<64, true, false>, grid, 128, 0, stream, q, kv, out, ws,
                  batch, heads, seq_len, chunk, qscale, q4, seq_lens);
    else
      rc = launch("decode_attention", decode_attn_kernel<64, false, false>, grid, 128, 0, stream, q, kv, out, ws,
                  batch, heads, seq_len, chunk, qscale, q4, seq_lens);
  }
  if (rc || splits == 1) return rc;
  if (head_dim == 128)
    return launch("decode_attention_combine", decode_attn_combine_kernel<128>, bh, 128, 0, stream, ws, out, heads, splits);
  return launch("decode_attention_combine", decode_attn_combine_kernel<64>, bh, 64, 0, stream, ws, out, heads, splits);
}

}  // namespace kvpr
