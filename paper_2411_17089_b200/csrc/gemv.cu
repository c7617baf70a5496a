// Small-batch decode projection on the CUDA cores: D[m, n] = epilogue(sum_k A[m, k] W[n, k]).
//
// At batch <= 8 a decode projection (out-proj, fc1, fc2, LM head) is a weight stream with
// almost no math: 2 bytes of W feed M <= 8 FMAs.  The tensor-core swap-AB kernel
// (gemm_tcgen05.cu) reaches HBM rate only once >= 140 CTAs stream, and small layers have
// far fewer 128-row weight tiles than that (OPT-125M shape: 6 tiles for out-proj and fc2),
// so their time is the per-CTA streaming rate plus the tcgen05 prologue (TMEM alloc,
// barrier init, descriptor prefetch): ~6 us for a 1.2 MB weight.  Here every warp streams
// its own slice with 16-byte non-allocating loads that are issued BEFORE the PDL wait
// (weights never depend on the previous kernel), so the weight fetch overlaps the previous
// kernel's tail and the whole matrix is in flight at once across the grid.
//
// Work split: a warp owns kNC consecutive output columns and one of KS k-slices; a CTA of
// 8 warps holds 8/KS column groups x KS slices.  KS is picked per shape so the grid covers
// the SMs.  Reduction order is fixed (lane-sequential FMAs, xor-shuffle tree, slices summed
// in slice order), so results are deterministic — but the k order differs from the tensor-core
// kernels, so this path is used only for projections whose outputs K1 never rebuilds
// (not the q/k/v projection; see kvpr_linear_ws in include/kvpr.h).

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {

namespace {

constexpr int kGemvWarps = 8;
constexpr int kNC = 2;  // output columns per warp
constexpr int kPF = 4;  // 16-byte units per lane and column issued before the PDL wait
constexpr int kLnVec = 2;  // LN prologue: float4 per thread per row held in registers (hidden <= 2048)

__device__ __forceinline__ uint4 ld_stream(const __half* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __half22float2(h[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}

// one 16-byte unit of K: acc[c][m] += W[n_c, 8u..8u+8) . A[m, 8u..8u+8), A from shared memory
template <int MP>
__device__ __forceinline__ void fma_unit(float (&acc)[kNC][MP], const uint4 (&wv)[kNC], const uint4* sa, int units,
                                         int M, int u) {
  float wf[kNC][8];
#pragma unroll
  for (int c = 0; c < kNC; ++c) unpack8(wv[c], wf[c]);
#pragma unroll
  for (int m = 0; m < MP; ++m) {
    if (m < M) {
      float af[8];
      unpack8(sa[m * units + u], af);
#pragma unroll
      for (int c = 0; c < kNC; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[c][m] = fmaf(wf[c][e], af[e], acc[c][m]);
    }
  }
}

// the tensor-core kernels' scalar epilogue for one output element (bias, scale, ReLU, segment scatter)
__device__ __forceinline__ void store_one(const GemmArgs& p, int m, int n, float v) {
  if (p.bias != nullptr) v += __half2float(p.bias[n]);
  if (n < p.scale_cols) v *= p.scale;
  if (p.flags & KVPR_EPI_RELU) v = fmaxf(v, 0.f);
  const int seg = n / p.seg_width;
  const int col = n - seg * p.seg_width;
  char* sp = static_cast<char*>(seg == 0 ? p.seg_ptr[0] : (seg == 1 ? p.seg_ptr[1] : p.seg_ptr[2]));
  const long long gs = seg == 0 ? p.seg_group_stride[0] : (seg == 1 ? p.seg_group_stride[1] : p.seg_group_stride[2]);
  const long long off = (m % p.row_group) * p.ld + (m / p.row_group) * gs + col;
  if (p.flags & KVPR_EPI_F32) {
    float* o = reinterpret_cast<float*>(sp) + off;
    *o = (p.flags & KVPR_EPI_ACCUM) ? *o + v : v;
  } else {
    reinterpret_cast<__half*>(sp)[off] = __float2half_rn(v);
  }
}

// LN-fused variant: A = LayerNorm(x) of fp32 rows, computed by every CTA into its staging buffer with
// layernorm_kernel's exact arithmetic (same thread -> column map, helpers, reduction tree), so A and
// the output carry the bits of the two-kernel LN -> projection sequence; CTA 0 also stores A to y
template <int MP, bool kLN>
__global__ void __launch_bounds__(kGemvWarps * 32)
    gemv_kernel(const __half* __restrict__ a, long long lda, const __half* __restrict__ w, long long ldw,
                const GemmArgs p, int ks_log2, const GemvLn ln) {
  extern __shared__ uint4 sa[];  // A staged once per CTA: [M][K/8] 16-byte units
  __shared__ float red[kGemvWarps][kNC * MP];
  pdl_trigger();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int KS = 1 << ks_log2;
  const int groups = kGemvWarps >> ks_log2;
  const int group = warp >> ks_log2;
  const int slice = warp & (KS - 1);
  const int n0 = (blockIdx.x * groups + group) * kNC;
  const int units = p.K >> 3;
  const int per = (units + KS - 1) / KS;
  const int u0 = slice * per;
  const int u1 = min(units, u0 + per);

  const __half* wr[kNC];
  bool live[kNC];
#pragma unroll
  for (int c = 0; c < kNC; ++c) {
    live[c] = n0 + c < p.N;
    wr[c] = w + static_cast<long long>(live[c] ? n0 + c : 0) * ldw;
  }

  // weights of the first kPF units per lane: issued before the wait (independent of earlier kernels)
  uint4 cur[kPF][kNC];
#pragma unroll
  for (int j = 0; j < kPF; ++j) {
    const int u = u0 + lane + 32 * j;
#pragma unroll
    for (int c = 0; c < kNC; ++c) cur[j][c] = (u < u1 && live[c]) ? ld_stream(wr[c] + u * 8) : make_uint4(0, 0, 0, 0);
  }
  pdl_wait();
  if constexpr (kLN) {
    // the rows are loaded once into registers (hidden <= 4 * 256 * kLnVec, checked on the host);
    // the passes then run from registers like layernorm_kernel's
    __shared__ float lnred[MP][kGemvWarps];
    __shared__ float lnstat[MP];
    const int nvec = p.K >> 2;
    float4 xv[MP][kLnVec];
#pragma unroll
    for (int m = 0; m < MP; ++m)
#pragma unroll
      for (int i = 0; i < kLnVec; ++i) {
        const int c = threadIdx.x + i * kGemvWarps * 32;
        xv[m][i] = (m < p.M && c < nvec) ? reinterpret_cast<const float4*>(ln.x + m * ln.ldx)[c]
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    float mean[MP], rstd[MP];
    // pass 1: row sums -> mean
#pragma unroll
    for (int m = 0; m < MP; ++m) {
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < kLnVec; ++i) a += ln_vec_sum(xv[m][i]);
      a = warp_sum(a);
      if (lane == 0) lnred[m][warp] = a;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int m = 0; m < MP; ++m) {
        const float t = warp_sum(lane < kGemvWarps ? lnred[m][lane] : 0.f);
        if (lane == 0) lnstat[m] = t;
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MP; ++m) mean[m] = lnstat[m] / p.K;
    __syncthreads();
    // pass 2: centred squares -> rstd
#pragma unroll
    for (int m = 0; m < MP; ++m) {
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < kLnVec; ++i)
        if (threadIdx.x + i * kGemvWarps * 32 < nvec) a += ln_vec_sq(xv[m][i], mean[m]);
      a = warp_sum(a);
      if (lane == 0) lnred[m][warp] = a;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int m = 0; m < MP; ++m) {
        const float t = warp_sum(lane < kGemvWarps ? lnred[m][lane] : 0.f);
        if (lane == 0) lnstat[m] = t;
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MP; ++m) rstd[m] = ln_rstd(lnstat[m], p.K, ln.eps);
    // normalise into the staging buffer (and y, from CTA 0)
    uint2* sa2 = reinterpret_cast<uint2*>(sa);
#pragma unroll
    for (int m = 0; m < MP; ++m) {
      if (m < p.M) {
#pragma unroll
        for (int i = 0; i < kLnVec; ++i) {
          const int c = threadIdx.x + i * kGemvWarps * 32;
          if (c < nvec) {
            const uint2 o = ln_vec_out(xv[m][i], mean[m], rstd[m], ln.gamma, ln.beta, c);
            sa2[m * nvec + c] = o;
            if (blockIdx.x == 0 && ln.y != nullptr) *reinterpret_cast<uint2*>(ln.y + m * ln.ldy + 4 * c) = o;
          }
        }
      }
    }
  } else {
    // A (written by the previous kernel): every 16-byte unit in flight at once, then shared memory
    for (int i = threadIdx.x; i < p.M * units; i += blockDim.x) {
      const int m = i / units;
      sa[i] = __ldg(reinterpret_cast<const uint4*>(a + m * lda) + (i - m * units));
    }
  }
  __syncthreads();

  float acc[kNC][MP];
#pragma unroll
  for (int c = 0; c < kNC; ++c)
#pragma unroll
    for (int m = 0; m < MP; ++m) acc[c][m] = 0.f;

  // software pipeline: the next kPF units' weights are issued before this batch's FMAs
  for (int ub = u0 + lane; ub < u1; ub += 32 * kPF) {
    uint4 nxt[kPF][kNC];
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
      const int u = ub + 32 * (kPF + j);
#pragma unroll
      for (int c = 0; c < kNC; ++c) nxt[j][c] = (u < u1 && live[c]) ? ld_stream(wr[c] + u * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
      const int u = ub + 32 * j;
      if (u < u1) fma_unit<MP>(acc, cur[j], sa, units, p.M, u);
    }
#pragma unroll
    for (int j = 0; j < kPF; ++j)
#pragma unroll
      for (int c = 0; c < kNC; ++c) cur[j][c] = nxt[j][c];
  }

  // warp tree, then slices in order
#pragma unroll
  for (int c = 0; c < kNC; ++c)
#pragma unroll
    for (int m = 0; m < MP; ++m) {
      float v = acc[c][m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[c][m] = v;
    }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < kNC; ++c)
#pragma unroll
      for (int m = 0; m < MP; ++m) red[warp][c * MP + m] = acc[c][m];
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < groups * kNC * MP) {
    const int g = t / (kNC * MP);
    const int idx = t - g * (kNC * MP);
    const int c = idx / MP;
    const int m = idx - c * MP;
    const int n = (blockIdx.x * groups + g) * kNC + c;
    if (m < p.M && n < p.N) {
      float v = 0.f;
      for (int s = 0; s < KS; ++s) v += red[g * KS + s][idx];
      store_one(p, m, n, v);
    }
  }
}

}  // namespace

int gemv_slices(int N, int device) {
  const int sms = sm_count(device);
  int ks_log2 = 0;
  while (ks_log2 < 3 && (N + kNC * (kGemvWarps >> ks_log2) - 1) / (kNC * (kGemvWarps >> ks_log2)) < sms) ++ks_log2;
  return ks_log2;
}

size_t gemv_smem_bytes(int M, int K) { return static_cast<size_t>(M) * K * 2; }

int gemv_f16(const void* a, long long lda, const void* w, long long ldw, const GemmArgs& args, cudaStream_t stream,
             const GemvLn* ln) {
  if (args.M < 1 || args.M > kGemvMaxM) {
    set_error("gemv: needs 1 <= M <= %d (M=%d)", kGemvMaxM, args.M);
    return KVPR_EINVAL;
  }
  const size_t smem = gemv_smem_bytes(args.M, args.K);
  if (smem > kGemvMaxSmem) {
    set_error("gemv: M*K*2 = %zu B of staged activations exceeds %d B", smem, kGemvMaxSmem);
    return KVPR_EINVAL;
  }
  if (ln != nullptr && (ln->x == nullptr || ln->gamma == nullptr || ln->beta == nullptr || ln->ldx % 4 != 0 ||
                        ln->ldy % 4 != 0 || args.K % 4 != 0 || args.K > kGemvLnMaxK)) {
    set_error("gemv: LayerNorm operands null, strides not multiples of 4, or hidden %d > %d", args.K, kGemvLnMaxK);
    return KVPR_EINVAL;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_done[64] = {0};
  if (dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(gemv_kernel<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvMaxSmem);
    cudaFuncSetAttribute(gemv_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvMaxSmem);
    cudaFuncSetAttribute(gemv_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvMaxSmem);
    cudaFuncSetAttribute(gemv_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvMaxSmem);
    attr_done[dev] = 1;
  }
  const int ks_log2 = gemv_slices(args.N, dev);
  const int cols_per_cta = kNC * (kGemvWarps >> ks_log2);
  const unsigned grid = static_cast<unsigned>((args.N + cols_per_cta - 1) / cols_per_cta);
  const __half* ap = static_cast<const __half*>(a);
  const __half* wp = static_cast<const __half*>(w);
  const GemvLn l = ln != nullptr ? *ln : GemvLn{};
  const unsigned thr = kGemvWarps * 32;
  if (ln != nullptr) {
    if (args.M <= 4) return launch("gemv_ln", gemv_kernel<4, true>, grid, thr, smem, stream, ap, lda, wp, ldw, args, ks_log2, l);
    return launch("gemv_ln", gemv_kernel<8, true>, grid, thr, smem, stream, ap, lda, wp, ldw, args, ks_log2, l);
  }
  if (args.M <= 4) return launch("gemv", gemv_kernel<4, false>, grid, thr, smem, stream, ap, lda, wp, ldw, args, ks_log2, l);
  return launch("gemv", gemv_kernel<8, false>, grid, thr, smem, stream, ap, lda, wp, ldw, args, ks_log2, l);
}

}  // namespace kvpr
