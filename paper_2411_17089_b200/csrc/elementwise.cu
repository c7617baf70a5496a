// Row kernels of the OPT decode layer: LayerNorm (K5), token + learned
// position embedding (K7) and the greedy argmax behind the LM head (K8).
// All are HBM/latency bound; rows map to CTAs, columns to 128-bit vectors.
//
// OPT semantics (not in the reference package, which has no decoder —
// SURVEY.md §8a note 2): pre-LN blocks, learned positions with offset 2,
// fp32 residual stream here (HF keeps fp16; fp32 is closer to the oracle).

#include <float.h>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {

namespace {

constexpr int kRowThreads = 256;

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

// one CTA per row; two-pass (mean, then centred variance) in fp32 from registers
template <int VPT>  // float4 vectors per thread
__global__ void __launch_bounds__(kRowThreads) layernorm_kernel(const float* __restrict__ x, long long ldx,
                                                                const __half* __restrict__ gamma,
                                                                const __half* __restrict__ beta, __half* __restrict__ out,
                                                                long long ldo, int hidden, float eps) {
  __shared__ float red[32];
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + row * ldx);
  const int nvec = hidden / 4;
  float4 v[VPT];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * kRowThreads;
    v[i] = (c < nvec) ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += ln_vec_sum(v[i]);
  }
  const float mean = block_sum(s, red) / hidden;
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * kRowThreads;
    if (c < nvec) ss += ln_vec_sq(v[i], mean);
  }
  const float rstd = ln_rstd(block_sum(ss, red), hidden, eps);
  __half* o = out + row * ldo;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * kRowThreads;
    if (c < nvec) *reinterpret_cast<uint2*>(o + 4 * c) = ln_vec_out(v[i], mean, rstd, gamma, beta, c);
  }
}

__global__ void embed_kernel(const int* __restrict__ tokens, const __half* __restrict__ tok_emb,
                             const __half* __restrict__ pos_emb, float* __restrict__ out, int batch, int pos_begin,
                             int hidden, int pos_offset) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const int pos = pos_begin + row / batch;
  const int tok = tokens[row];
  const __half2* e = reinterpret_cast<const __half2*>(tok_emb + (long long)tok * hidden);
  const __half2* p = reinterpret_cast<const __half2*>(pos_emb + (long long)(pos + pos_offset) * hidden);
  float2* o = reinterpret_cast<float2*>(out + (long long)row * hidden);
  for (int c = threadIdx.x; c < hidden / 2; c += blockDim.x) {
    const float2 a = __half22float2(e[c]), b = __half22float2(p[c]);
    o[c] = make_float2(a.x + b.x, a.y + b.y);
  }
}

// one CTA per row; ties resolve to the smallest index (numpy/torch argmax convention).
// 16-byte loads, four in flight per thread: a 50272-wide fp32 row is ~200 KB, streamed at
// the SM's load bandwidth instead of one dependent scalar load per thread per iteration.
constexpr int kArgmaxThreads = 1024;

__device__ __forceinline__ void amax_take(float v, int c, float& best, int& bi) {
  if (v > best || (v == best && c < bi)) {
    best = v;
    bi = c;
  }
}

__global__ void __launch_bounds__(kArgmaxThreads) argmax_kernel(const float* __restrict__ logits, long long ld,
                                                                int cols, int* __restrict__ out_idx,
                                                                float* __restrict__ out_val) {
  __shared__ float sv[32];
  __shared__ int si[32];
  pdl_trigger();
  pdl_wait();
  const float* r = logits + blockIdx.x * ld;
  float best = -FLT_MAX;
  int bi = 0x7fffffff;
  const bool vec = ((reinterpret_cast<uintptr_t>(r) & 15) == 0);
  const int nv = vec ? cols / 4 : 0;
  const float4* r4 = reinterpret_cast<const float4*>(r);
  int c = threadIdx.x;
  for (; c + 3 * kArgmaxThreads < nv; c += 4 * kArgmaxThreads) {
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldg(r4 + c + u * kArgmaxThreads);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b0 = 4 * (c + u * kArgmaxThreads);
      amax_take(x[u].x, b0, best, bi);
      amax_take(x[u].y, b0 + 1, best, bi);
      amax_take(x[u].z, b0 + 2, best, bi);
      amax_take(x[u].w, b0 + 3, best, bi);
    }
  }
  for (; c < nv; c += kArgmaxThreads) {
    const float4 x = __ldg(r4 + c);
    amax_take(x.x, 4 * c, best, bi);
    amax_take(x.y, 4 * c + 1, best, bi);
    amax_take(x.z, 4 * c + 2, best, bi);
    amax_take(x.w, 4 * c + 3, best, bi);
  }
  for (int t = 4 * nv + threadIdx.x; t < cols; t += kArgmaxThreads) amax_take(r[t], t, best, bi);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    amax_take(ov, oi, best, bi);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    best = (l < nw) ? sv[l] : -FLT_MAX;
    bi = (l < nw) ? si[l] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      amax_take(ov, oi, best, bi);
    }
    if (threadIdx.x == 0) {
      out_idx[blockIdx.x] = bi;
      if (out_val) out_val[blockIdx.x] = best;
    }
  }
}

}  // namespace

int layernorm(const float* x, long long ldx, const __half* gamma, const __half* beta, __half* out, long long ldo,
              int rows, int hidden, float eps, cudaStream_t stream) {
  if (rows < 0 || hidden <= 0 || hidden % 4 != 0 || ldx % 4 != 0 || ldo % 4 != 0) {
    set_error("layernorm: rows=%d hidden=%d ldx=%lld ldo=%lld (hidden, strides must be multiples of 4)", rows, hidden,
              ldx, ldo);
    return KVPR_EINVAL;
  }
  if (rows == 0) return KVPR_OK;
  const int nvec = hidden / 4;
  const int vpt = (nvec + kRowThreads - 1) / kRowThreads;
  if (vpt <= 1)
    return launch("layernorm", layernorm_kernel<1>, rows, kRowThreads, 0, stream, x, ldx, gamma, beta, out, ldo, hidden, eps);
  else if (vpt <= 2)
    return launch("layernorm", layernorm_kernel<2>, rows, kRowThreads, 0, stream, x, ldx, gamma, beta, out, ldo, hidden, eps);
  else if (vpt <= 4)
    return launch("layernorm", layernorm_kernel<4>, rows, kRowThreads, 0, stream, x, ldx, gamma, beta, out, ldo, hidden, eps);
  else if (vpt <= 8)
    return launch("layernorm", layernorm_kernel<8>, rows, kRowThreads, 0, stream, x, ldx, gamma, beta, out, ldo, hidden, eps);
  else {
    set_error("layernorm: hidden=%d too large (max 8192)", hidden);
    return KVPR_EINVAL;
  }
}

int embed(const int* tokens, const __half* tok_emb, const __half* pos_emb, float* out, int rows, int batch,
          int pos_begin, int hidden, int pos_offset, cudaStream_t stream) {
  if (rows < 0 || batch <= 0 || hidden <= 0 || hidden % 2 != 0 || pos_begin < 0) {
    set_error("embed: bad shape rows=%d batch=%d hidden=%d pos_begin=%d", rows, batch, hidden, pos_begin);
    return KVPR_EINVAL;
  }
  if (rows == 0) return KVPR_OK;
  return launch("embed", embed_kernel, rows, 256, 0, stream, tokens, tok_emb, pos_emb, out, batch, pos_begin, hidden,
                pos_offset);
}

int argmax_rows(const float* logits, long long ld, int rows, int cols, int* out_idx, float* out_val,
                cudaStream_t stream) {
  if (rows < 0 || cols <= 0 || ld < cols) {
    set_error("argmax: bad shape rows=%d cols=%d ld=%lld", rows, cols, ld);
    return KVPR_EINVAL;
  }
  if (rows == 0) return KVPR_OK;
  return launch("argmax", argmax_kernel, rows, kArgmaxThreads, 0, stream, logits, ld, cols, out_idx, out_val);
}

}  // namespace kvpr
