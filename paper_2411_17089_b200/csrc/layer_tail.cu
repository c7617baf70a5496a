// Fused small-batch decode layer tail: K2 -> out-proj + residual -> LN2 -> fc1 + ReLU -> fc2 +
// residual [-> LayerNorm of the new residual] in ONE cooperative kernel.
//
// At batch <= 8 on a small model (BASELINE config 1: OPT-125M shape, b4) a decode layer moves
// ~14 MB of weights and ~3 MB of KV: every kernel of the chain is a few microseconds of launch,
// ramp and drain around well under a microsecond of streaming, and the chain of dependent launches,
// not PCIe, set the step time (round-2 sweep: with no PCIe on the path at all the multi-kernel layer
// still took ~40 us; profiles/r02_c1_modes.jsonl has the unfused chain beside this kernel).  Here the
// steps after the q/k/v projection run as stages of one grid (one CTA per SM) separated by grid-wide
// barriers (~1 us each) instead of kernel boundaries:
//
//   entry  each CTA bulk-copies ITS weight rows of all three projections (CTA c owns output columns
//          [cN/G, (c+1)N/G) of each) into shared memory, so the weight stream runs under stage A
//   A  split-KV attention over the merged pages (numerics.decode_attention, numerics.py:166-191):
//      (sequence, head, split) items, the K2 sweep (attn_common.cuh); softmax states to ws
//   B  every CTA merges the split states in split order (K2's combine) into its staging rows, then
//      out-proj + bias + residual for its columns
//   C  LN2 (every CTA normalises the rows itself) + fc1 + bias + ReLU
//   D  fc2 + bias + residual
//   E  the last CTA to arrive normalises the new residual (optional): the next layer's LN1 straight
//      into its X slot, or the final LN before the LM head
//
// The projections are tiny per CTA (6-21 weight rows x 4 activation rows), so they run on the warp
// tensor-core path (mma.sync m16n8k16, fp32 accumulate, operands by ldmatrix from padded rows),
// K split over the 8 warps and the warp partials summed in warp order.  Deterministic (fixed
// orders, no atomics on data), but not the multi-kernel path's summation order: results agree with
// it to fp32 rounding, not bit for bit.  Never used for the q/k/v projection (its k, v must carry
// K1's bits).  The grid barrier needs every CTA resident: launched cooperatively, one CTA per SM,
// and the PDL trigger fires only after the first barrier (all CTAs resident), so a dependent kernel
// cannot take an SM this grid still needs.

#include <stdlib.h>

#include <map>
#include <mutex>

#include "attn_common.cuh"
#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {

namespace {

using namespace attn;

constexpr int kTailThreads = 256;
constexpr int kTailWarps = kTailThreads / 32;
constexpr int kTailSyncWords = 64;    // per (device, stream): a 64-bit arrival counter (+ padding)
constexpr int kTailRounds = 4;        // grid barriers per launch (every CTA arrives once at each)
constexpr int kTailMaxTiles = 2;      // 16-row weight tiles per CTA and projection (<= 32 columns per CTA)
constexpr size_t kTailSmemBudget = 221 * 1024;

// KVPR_GEMM_TRACE builds (tools/tail_bench.py): per-CTA globaltimer stamps at the stage boundaries
__device__ unsigned long long* g_tail_trace = nullptr;
__device__ __forceinline__ void tstamp(int slot) {
#ifdef KVPR_GEMM_TRACE
  if (threadIdx.x == 0 && g_tail_trace != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tail_trace[blockIdx.x * 24 + slot] = t;
  }
#else
  (void)slot;
#endif
}

struct TailParams {
  int M, H, heads, F, S;
  float qscale, eps;
  const __half* q;
  const __half* kv;
  __half* attn;
  const __half* wo;
  const __half* bo;
  float* hres;
  const __half* ln2_g;
  const __half* ln2_b;
  const __half* w1;
  const __half* b1;
  __half* mid;
  const __half* w2;
  const __half* b2;
  const __half* lnx_g;  // optional stage E: LayerNorm of the new residual -> lnx_out
  const __half* lnx_b;
  __half* lnx_out;
  long long lnx_ld;
  const __half* wq;     // optional with stage E: the next layer's [W_q; W_k; W_v] [3H][H] and bias
  const __half* bq;
  __half* q_out;        // its q [M][H]
  __half* page_out;     // its k, v page: K [M][H] then V [M][H]
  const __half* kv_alt;  // optional: attention positions [alt_lo, alt_hi) read from here (host store, same layout)
  int alt_lo, alt_hi;
  int alt_npos;          // > 0: each item's part of [alt_lo, alt_hi) (<= alt_npos positions) is pulled into
                         // shared memory at kernel entry (under the prologue); 0: read in place
  __half* x_store;       // optional: the normalised rows also here (host X store row of the next unit)
  __half* page_store;    // optional: the next layer's k, v page also here (host KV store page)
  float* part;                 // attention split partials [pairs * splits][D + 4] (m, l, pad, pad, acc[D])
  unsigned long long* count;   // library-owned monotone arrival counter (kTailRounds * G per launch)
  int splits, chunk;
  int nh, nf;                  // max columns per CTA of the hidden-wide / ffn-wide projections
};

__device__ __forceinline__ void prefetch_l2(const void* p, long long bytes) {
  while (bytes > 0) {
    const unsigned n = static_cast<unsigned>(bytes > (1ll << 30) ? (1ll << 30) : bytes);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(n) : "memory");
    p = static_cast<const char*>(p) + n;
    bytes -= n;
  }
}

// 1-D bulk copy global -> this CTA's shared memory, completion counted on `bar` (16-byte aligned spans)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// rows [M][K] fp16 global (written earlier in this grid: read through L2) -> shared rows of stride
// ldk, U 16-byte loads in flight per thread before the first store (a load -> store loop would pay
// one L2 round trip per iteration)
template <int U>
__device__ __forceinline__ void rows_g2s(__half* dst, int ldk, const __half* src, int M, int K) {
  const int per_row = K >> 3, n16 = M * per_row;
  const uint4* g = reinterpret_cast<const uint4*>(src);
  for (int i0 = threadIdx.x; i0 < n16; i0 += U * kTailThreads) {
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = i0 + j * kTailThreads;
      if (i < n16) r[j] = __ldcg(g + i);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = i0 + j * kTailThreads;
      if (i < n16) {
        const int m = i / per_row;
        reinterpret_cast<uint4*>(dst + static_cast<long long>(m) * ldk)[i - m * per_row] = r[j];
      }
    }
  }
}

// Grid barrier on a monotone 64-bit counter: the CTA's writes are ordered before thread 0's release
// arrival by the bar.sync (release is cumulative), the acquire poll orders everything after it.  No
// fence, no reset, no return value on the arrival: one fire-and-forget reduction and one polling
// round trip.  target = base + k * G for the k-th barrier of this launch.
__device__ __forceinline__ void grid_barrier(unsigned long long* count, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
    unsigned long long cur;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(count) : "memory");
    } while (cur < target);
  }
  __syncthreads();
}

// LayerNorm of one fp32 row by one warp, two-pass (mean, then centred variance) like
// layernorm_kernel; the row is read through L2 (written earlier in this grid); fp16 out
__device__ __forceinline__ void warp_layernorm_row(const float* x, int H, const __half* gamma, const __half* beta,
                                                   float eps, __half* out) {
  constexpr int VW = 8;  // float4 per lane: H <= 1024
  const int lane = threadIdx.x & 31;
  const int nvec = H >> 2;
  float4 v[VW];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VW; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < nvec ? __ldcg(reinterpret_cast<const float4*>(x) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    s += ln_vec_sum(v[i]);
  }
  const float mean = warp_sum(s) / H;
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VW; ++i)
    if (lane + 32 * i < nvec) ss += ln_vec_sq(v[i], mean);
  const float rstd = ln_rstd(warp_sum(ss), H, eps);
#pragma unroll
  for (int i = 0; i < VW; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) *reinterpret_cast<uint2*>(out + 4 * c) = ln_vec_out(v[i], mean, rstd, gamma, beta, c);
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}

__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// Projection columns [n0, n1) of this CTA on the warp tensor cores: out(m, n) = sum_k A[m, k] W[n, k]
// with this CTA's weight rows sw [16 * tiles][ldk] (row n - n0) and the activation rows sa [8][ldk]
// (rows >= M are don't-care: they only feed output columns that are never stored) in shared memory.
// D^T = W A^T: the 16-row weight tiles are the MMA's M, the 8 activation rows its N.  Warp w takes
// the k-steps w, w + 8, ... of every tile; the 8 warp partials meet in `red` and are summed in warp
// order by one thread per output.  ldk = K + 8 halves: the 8 rows of an ldmatrix hit distinct banks.
template <class Epi>
__device__ __forceinline__ void proj_mma(const __half* sa, const __half* sw, int ldk, int M, int K, int n0, int n1,
                                         float* red, Epi epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = n1 - n0;
  const int tiles = (rows + 15) >> 4;
  const int ksteps = K >> 4;
  float acc[kTailMaxTiles][4];
#pragma unroll
  for (int t = 0; t < kTailMaxTiles; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[t][i] = 0.f;
  // ldmatrix row addresses: A (weights) x4 = rows (lane % 8) + 8 ((lane / 8) % 2), k + 8 (lane / 16);
  // B (activations) x2 = rows lane % 8, k + 8 ((lane / 8) % 2).  Rows past the live ones re-read row 0:
  // they only feed accumulator rows / columns that are never stored
  uint32_t a_base[kTailMaxTiles];
#pragma unroll
  for (int t = 0; t < kTailMaxTiles; ++t) {
    const int r = t * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
    a_base[t] = smem_u32(sw + (r < rows ? r : 0) * ldk + (lane >> 4) * 8);
  }
  const int rb = lane & 7;
  const uint32_t b_base = smem_u32(sa + (rb < M ? rb : 0) * ldk + ((lane >> 3) & 1) * 8);
  for (int ks = warp; ks < ksteps; ks += kTailWarps) {
    uint32_t b[2];
    ldsm_x2(b_base + ks * 32, b);
#pragma unroll
    for (int t = 0; t < kTailMaxTiles; ++t) {
      if (t < tiles) {
        uint32_t a[4];
        ldsm_x4(a_base[t] + ks * 32, a);
        mma_16816(acc[t], a, b);
      }
    }
  }
  // D fragment: (row g, cols 2q, 2q+1) and (row g + 8, same cols), g = lane / 4, q = lane % 4;
  // row = weight row (output column n), col = activation row m
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int t = 0; t < kTailMaxTiles; ++t) {
    if (t < tiles) {
      float* r = red + ((warp * kTailMaxTiles + t) * 16) * 8;
      r[g * 8 + 2 * q] = acc[t][0];
      r[g * 8 + 2 * q + 1] = acc[t][1];
      r[(g + 8) * 8 + 2 * q] = acc[t][2];
      r[(g + 8) * 8 + 2 * q + 1] = acc[t][3];
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < tiles * 16 * 8; o += kTailThreads) {
    const int t = o >> 7, row = (o >> 3) & 15, m = o & 7;
    const int n = n0 + t * 16 + row;
    if (m < M && n < n1) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kTailWarps; ++w) v += red[((w * kTailMaxTiles + t) * 16 + row) * 8 + m];
      epi(m, n, v);
    }
  }
}

// The same product with the tcgen05 kernels' k order -- one accumulator per element, k ascending in
// 16-wide steps, no K split -- which mma.sync reproduces bit for bit (tests/test_layer_tail_gpu.py,
// tools/mma_bits_probe.py).  For the q/k/v projection, whose k, v must equal K1's rebuild.  Warp t
// takes tile t.
template <class Epi>
__device__ __forceinline__ void proj_mma_kseq(const __half* sa, const __half* sw, int ldk, int M, int K, int n0,
                                              int n1, Epi epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = n1 - n0;
  const int tiles = (rows + 15) >> 4;
  if (warp >= tiles) return;
  const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const uint32_t a_base = smem_u32(sw + (r < rows ? r : 0) * ldk + (lane >> 4) * 8);
  const int rb = lane & 7;
  const uint32_t b_base = smem_u32(sa + (rb < M ? rb : 0) * ldk + ((lane >> 3) & 1) * 8);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int ks = 0; ks < (K >> 4); ++ks) {
    uint32_t a[4], b[2];
    ldsm_x4(a_base + ks * 32, a);
    ldsm_x2(b_base + ks * 32, b);
    mma_16816(acc, a, b);
  }
  const int g = lane >> 2, q = lane & 3;
  const int na = n0 + warp * 16 + g, nb = na + 8, m0 = 2 * q;
  if (na < n1) {
    if (m0 < M) epi(m0, na, acc[0]);
    if (m0 + 1 < M) epi(m0 + 1, na, acc[1]);
  }
  if (nb < n1) {
    if (m0 < M) epi(m0, nb, acc[2]);
    if (m0 + 1 < M) epi(m0 + 1, nb, acc[3]);
  }
}

// Shared-memory carve-up (bytes, 16-aligned).  This CTA's weight rows (row stride K + 8 halves);
// the activation rows of stages B / C ([M][H + 8]) with the attention partials behind them, both
// overlaid by stage D's [M][F + 8] rows; the MMA warp partials; this CTA's residual columns; the
// LayerNorm rows and this CTA's biases.
struct TailSmem {
  uint32_t wo, w1, w2, wq, act, part, red, res, prm, host, total;
};

__host__ __device__ inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// q/k/v columns per CTA (whole 8-column units): the most any CTA of a G-CTA grid owns
__host__ __device__ inline int tail_nq(int H, int G) { return 8 * ((3 * H / 8 + G - 1) / G); }

__host__ __device__ inline TailSmem tail_smem(int M, int H, int F, int nh, int nf, int nq, int items, int D,
                                              uint32_t host_bytes = 0) {
  TailSmem t;
  t.wo = 0;
  t.w1 = t.wo + align16(static_cast<uint32_t>(nh) * (H + 8) * 2);
  t.w2 = t.w1 + align16(static_cast<uint32_t>(nf) * (H + 8) * 2);
  t.wq = t.w2 + align16(static_cast<uint32_t>(nh) * (F + 8) * 2);
  t.act = t.wq + align16(static_cast<uint32_t>(nq) * (H + 8) * 2);
  t.part = t.act + align16(static_cast<uint32_t>(M) * (H + 8) * 2);
  const uint32_t bc = t.part + align16(static_cast<uint32_t>(items) * (D + 4) * 4);
  const uint32_t d = t.act + align16(static_cast<uint32_t>(M) * (F + 8) * 2);
  t.red = bc > d ? bc : d;
  t.res = t.red + align16(kTailWarps * kTailMaxTiles * 16 * 8 * 4);
  t.prm = t.res + align16(static_cast<uint32_t>(M) * nh * 4);
  t.host = t.prm + align16(static_cast<uint32_t>(4 * H + 2 * nh + nf + nq) * 2);
  t.total = t.host + align16(host_bytes);
  return t;
}

template <int D>
__global__ void __launch_bounds__(kTailThreads, 1) layer_tail_kernel(const TailParams p) {
  constexpr int LPP = D / 8;
  constexpr int PPW = 32 / LPP;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t wbar[4];
  __shared__ float sm_m[kTailWarps], sm_l[kTailWarps];
  __shared__ float sm_acc[kTailWarps][D];
  __shared__ int s_flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  const int H = p.H, F = p.F, M = p.M;
  const int h0 = c * H / G, h1 = (c + 1) * H / G;  // 32-bit: H, F <= 4736, G <= 1024
  const int f0 = c * F / G, f1 = (c + 1) * F / G;
  // q/k/v columns in whole 8-column units (16-byte stores of the new page and its host copy)
  const int q0 = p.wq != nullptr ? 8 * (c * (3 * H / 8) / G) : 0, q1 = p.wq != nullptr ? 8 * ((c + 1) * (3 * H / 8) / G) : 0;
  const int nq = tail_nq(H, G);
  const int pairs = M * p.heads, items = pairs * p.splits;
  const int per_cta = (items + G - 1) / G;
  const TailSmem L = tail_smem(M, H, F, p.nh, p.nf, nq, items, D,
                               static_cast<uint32_t>(per_cta * p.alt_npos * 2 * D * 2));
  const int ldh = H + 8, ldf = F + 8;  // padded row strides (halves): conflict-free ldmatrix
  __half* sWo = reinterpret_cast<__half*>(smem + L.wo);
  __half* sW1 = reinterpret_cast<__half*>(smem + L.w1);
  __half* sW2 = reinterpret_cast<__half*>(smem + L.w2);
  __half* sWq = reinterpret_cast<__half*>(smem + L.wq);
  __half* sA = reinterpret_cast<__half*>(smem + L.act);
  float* sP = reinterpret_cast<float*>(smem + L.part);
  float* sRed = reinterpret_cast<float*>(smem + L.red);
  float* sR = reinterpret_cast<float*>(smem + L.res);  // [M][nh]: this CTA's residual columns
  __half* sG2 = reinterpret_cast<__half*>(smem + L.prm);  // LN2 gamma, beta; output-LN gamma, beta: [H] each
  __half* sBe2 = sG2 + H;                                  // (H % 8 == 0: every row 16-byte aligned)
  __half* sGx = sBe2 + H;
  __half* sBx = sGx + H;
  __half* sBo = sBx + H;
  __half* sB2 = sBo + p.nh;
  __half* sB1 = sB2 + p.nh;
  __half* sBq = sB1 + p.nf;
  __half* sH = reinterpret_cast<__half*>(smem + L.host);  // [per_cta][alt_npos][K, V][D]: host tail copy

  tstamp(0);
  // this CTA's weight rows of the three projections -> shared memory (one bulk copy per row, so the
  // rows land at the padded stride), under the attention stage
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < 4; ++i) mbar_init(&wbar[i], 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(&wbar[0], static_cast<uint32_t>(h1 - h0) * H * 2);
      mbar_arrive_expect_tx(&wbar[1], static_cast<uint32_t>(f1 - f0) * H * 2);
      mbar_arrive_expect_tx(&wbar[2], static_cast<uint32_t>(h1 - h0) * F * 2);
      mbar_arrive_expect_tx(&wbar[3], static_cast<uint32_t>(q1 - q0) * H * 2);
    }
    __syncwarp();
    for (int r = lane; r < h1 - h0; r += 32) {
      bulk_g2s(sWo + r * ldh, p.wo + static_cast<long long>(h0 + r) * H, H * 2, &wbar[0]);
      bulk_g2s(sW2 + r * ldf, p.w2 + static_cast<long long>(h0 + r) * F, F * 2, &wbar[2]);
    }
    for (int r = lane; r < f1 - f0; r += 32)
      bulk_g2s(sW1 + r * ldh, p.w1 + static_cast<long long>(f0 + r) * H, H * 2, &wbar[1]);
    for (int r = lane; r < q1 - q0; r += 32)
      bulk_g2s(sWq + r * ldh, p.wq + static_cast<long long>(q0 + r) * H, H * 2, &wbar[3]);
  }
  // small parameters (never written by a kernel), every load in flight before the first store:
  // LayerNorm rows as 16-byte units, this CTA's biases as scalars
  {
    const int u = H >> 3;  // 16-byte units per LayerNorm row
    const uint4* src[4] = {reinterpret_cast<const uint4*>(p.ln2_g), reinterpret_cast<const uint4*>(p.ln2_b),
                           reinterpret_cast<const uint4*>(p.lnx_out != nullptr ? p.lnx_g : p.ln2_g),
                           reinterpret_cast<const uint4*>(p.lnx_out != nullptr ? p.lnx_b : p.ln2_b)};
    uint4 v[2][4];
    __half bv[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int i = threadIdx.x + j * kTailThreads;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (i < u) v[j][r] = __ldg(src[r] + i);
      // biases in smem order: b_o, b_2 (this CTA's hidden columns), b_1, b_qkv
      const int nh2 = 2 * (h1 - h0), nb = nh2 + (f1 - f0) + (q1 - q0);
      if (i < nb)
        bv[j] = i < h1 - h0 ? p.bo[h0 + i]
                            : (i < nh2 ? p.b2[h0 + i - (h1 - h0)]
                                       : (i < nh2 + (f1 - f0) ? p.b1[f0 + i - nh2] : p.bq[q0 + i - nh2 - (f1 - f0)]));
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int i = threadIdx.x + j * kTailThreads;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (i < u) reinterpret_cast<uint4*>(sG2 + r * H)[i] = v[j][r];
      const int nh2 = 2 * (h1 - h0), nb = nh2 + (f1 - f0) + (q1 - q0);
      if (i < nb)
        (i < h1 - h0 ? sBo[i]
                     : (i < nh2 ? sB2[i - (h1 - h0)] : (i < nh2 + (f1 - f0) ? sB1[i - nh2] : sBq[i - nh2 - (f1 - f0)]))) = bv[j];
    }
  }
  // the transferred tail KV[l:s'-1] of this CTA's attention items, host store -> shared memory, every
  // load in flight at once: the PCIe round trip hides under the prologue (the host store was written by
  // earlier steps, stream-ordered before this launch)
  if (p.alt_npos > 0) {
    const int dl = D / 8;  // 16-byte units per K (or V) row of one head
    const int per_item = p.alt_npos * 2 * dl;
    const int total = per_cta * per_item;
    const long long page_stride = 2LL * M * H;
    for (int i0 = threadIdx.x; i0 < total; i0 += 4 * kTailThreads) {
      uint4 v[4];
      int dst[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + j * kTailThreads;
        dst[j] = -1;
        if (i < total) {
          const int k = i / per_item, r = i - k * per_item;
          const int pi = r / (2 * dl), kvu = r - pi * 2 * dl;
          const int it = c + k * G;
          if (it < items) {
            const int pair = it / p.splits, split = it - pair * p.splits;
            const int b = pair / p.heads, hd = pair - b * p.heads;
            const int lo = max(split * p.chunk, p.alt_lo), hi = min(min(p.S, split * p.chunk + p.chunk), p.alt_hi);
            if (lo + pi < hi) {
              const int kv = kvu / dl, uu = kvu - kv * dl;
              v[j] = *reinterpret_cast<const uint4*>(p.kv_alt + (lo + pi) * page_stride + static_cast<long long>(kv) * M * H +
                                                     static_cast<long long>(b) * H + hd * D + uu * 8);
              dst[j] = i;
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (dst[j] >= 0) reinterpret_cast<uint4*>(sH)[dst[j]] = v[j];
    }
  }
  pdl_wait();  // q, the pages and the residual come from the preceding kernels (and every earlier
               // launch's arrivals have landed: read the counter only after this)
  tstamp(1);
  // arrivals of this launch start at base: every launch adds exactly kTailRounds * G, every earlier
  // launch is complete after pdl_wait, and no CTA passes barrier 1 before every CTA has arrived, so
  // every CTA reads a value in [base, base + G)
  unsigned long long seen;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(p.count) : "memory");
  const unsigned long long round = static_cast<unsigned long long>(kTailRounds) * G;
  const unsigned long long base = seen - seen % round;
  if (threadIdx.x < M * (h1 - h0)) {
    const int m = threadIdx.x / (h1 - h0), n = h0 + threadIdx.x % (h1 - h0);
    sR[m * p.nh + (n - h0)] = p.hres[static_cast<long long>(m) * H + n];
  }

  __syncthreads();  // the host tail copy (sH) and the residual columns (sR) are in shared memory

  // ---------------- A: split-KV attention, partial softmax states to ws ----------------
  {
    const int glane = lane % LPP, grp = lane / LPP;
    const long long page_stride = 2LL * M * H;
    for (int it = c; it < items; it += G) {
      const int pair = it / p.splits, split = it - pair * p.splits;
      const int b = pair / p.heads, hd = pair - b * p.heads;
      const int p_lo = split * p.chunk, p_hi = min(p.S, p_lo + p.chunk);
      float q8[8];
      load8(p.q + static_cast<long long>(b) * H + hd * D + glane * 8, q8);
#pragma unroll
      for (int i = 0; i < 8; ++i) q8[i] *= p.qscale;
      Softmax8 st;
      st.init();
      if (p.kv_alt != nullptr && p_lo < p.alt_hi && p_hi > p.alt_lo) {  // this split reaches into the host tail
        const int lo = max(p_lo, p.alt_lo);
        AltSrc alt;
        alt.lo = lo;
        alt.hi = min(p_hi, p.alt_hi);
        if (p.alt_npos > 0) {  // the copy pulled at entry
          alt.base = sH + ((it - c) / G) * p.alt_npos * 2 * D;
          alt.stride = 2 * D;
          alt.v_off = D;
        } else {  // in place, over PCIe
          alt.base = p.kv_alt + lo * page_stride + static_cast<long long>(b) * H + hd * D;
          alt.stride = static_cast<int>(page_stride);
          alt.v_off = M * H;
        }
        sweep<D, 4, false, true>(p.kv + static_cast<long long>(b) * H + hd * D, page_stride,
                                 static_cast<long long>(M) * H, p_lo + warp * PPW, p_hi, kTailWarps * PPW, grp, q8,
                                 glane, st, nullptr, &alt);
      } else {
        sweep<D, 4>(p.kv + static_cast<long long>(b) * H + hd * D, page_stride, static_cast<long long>(M) * H,
                    p_lo + warp * PPW, p_hi, kTailWarps * PPW, grp, q8, glane, st);
      }
      merge_in_warp<LPP>(st);
      if (lane < LPP) {
        if (lane == 0) {
          sm_m[warp] = st.m;
          sm_l[warp] = st.l;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) sm_acc[warp][glane * 8 + i] = st.acc[i];
      }
      __syncthreads();
      if (threadIdx.x < D) {
        float m = -INFINITY, l = 0.f, a = 0.f;
#pragma unroll
        for (int w = 0; w < kTailWarps; ++w) m = fmaxf(m, sm_m[w]);
#pragma unroll
        for (int w = 0; w < kTailWarps; ++w) {
          const float f = (sm_m[w] == -INFINITY) ? 0.f : exp2f(sm_m[w] - m);
          l += sm_l[w] * f;
          a += sm_acc[w][threadIdx.x] * f;
        }
        float* w = p.part + static_cast<long long>(it) * (D + 4);
        w[4 + threadIdx.x] = a;
        if (threadIdx.x == 0) {
          w[0] = m;
          w[1] = l;
        }
      }
      __syncthreads();  // sm_* reused by the next item
    }
  }
  tstamp(2);
  grid_barrier(p.count, base + G);
  tstamp(3);
  pdl_trigger();  // every CTA of this grid is resident: a dependent grid may now take free SMs

  // ---------------- B: merge the splits (every CTA), out-proj + bias + residual ----------------
  {
    rows_g2s<12>(reinterpret_cast<__half*>(sP), 0, reinterpret_cast<const __half*>(p.part), 1, items * (D + 4) * 2);
    __syncthreads();
    tstamp(16);
    // split merge in split order (K2's combine): per (sequence, head) the split weights
    // f_s = 2^(m_s - max m) once, then every element sums acc_s * f_s / sum_s l_s f_s
    float* sF = sRed;  // scratch until the first projection: [pairs][splits] weights, [pairs] 1 / l
    float* sInvL = sRed + items;
    for (int pr = threadIdx.x; pr < pairs; pr += kTailThreads) {
      const float* w0 = sP + pr * p.splits * (D + 4);
      float mm = -INFINITY;
      for (int s2 = 0; s2 < p.splits; ++s2) mm = fmaxf(mm, w0[s2 * (D + 4)]);
      float ll = 0.f;
      for (int s2 = 0; s2 < p.splits; ++s2) {
        const float ms = w0[s2 * (D + 4)];
        const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - mm);
        sF[pr * p.splits + s2] = f;
        ll += w0[s2 * (D + 4) + 1] * f;
      }
      sInvL[pr] = ll;
    }
    __syncthreads();
    for (int e2 = threadIdx.x; e2 < (M * H) >> 1; e2 += kTailThreads) {
      const int e = 2 * e2;
      const int pr = e / D, dd = e - pr * D;  // pairs are (sequence, head) row-major: e indexes attn[m][e % H]
      const float* w0 = sP + pr * p.splits * (D + 4) + 4 + dd;
      float a0 = 0.f, a1 = 0.f;
      for (int s2 = 0; s2 < p.splits; ++s2) {
        const float f = sF[pr * p.splits + s2];
        const float2 v = *reinterpret_cast<const float2*>(w0 + s2 * (D + 4));
        a0 += v.x * f;
        a1 += v.y * f;
      }
      const float ll = sInvL[pr];
      const __half2 o = __floats2half2_rn(a0 / ll, a1 / ll);
      const int m = e / H;
      *reinterpret_cast<__half2*>(sA + m * ldh + (e - m * H)) = o;
      if (c == 0) *reinterpret_cast<__half2*>(p.attn + e) = o;
    }
    __syncthreads();
    tstamp(10);
    mbar_wait(&wbar[0], 0);
    tstamp(11);
    proj_mma(sA, sWo, ldh, M, H, h0, h1, sRed, [&](int m, int n, float v) {
      float* r = sR + m * p.nh + (n - h0);
      const float x = *r + (v + __half2float(sBo[n - h0]));
      *r = x;
      p.hres[static_cast<long long>(m) * H + n] = x;
    });
  }
  tstamp(4);
  grid_barrier(p.count, base + 2ull * G);
  tstamp(5);

  // ---------------- C: LN2 (every CTA) + fc1 + bias + ReLU ----------------
  for (int r = warp; r < M; r += kTailWarps)
    warp_layernorm_row(p.hres + static_cast<long long>(r) * H, H, sG2, sBe2, p.eps, sA + r * ldh);
  __syncthreads();
  tstamp(12);
  mbar_wait(&wbar[1], 0);
  tstamp(13);
  proj_mma(sA, sW1, ldh, M, H, f0, f1, sRed, [&](int m, int n, float v) {
    p.mid[static_cast<long long>(m) * F + n] = __float2half_rn(fmaxf(v + __half2float(sB1[n - f0]), 0.f));
  });
  tstamp(6);
  grid_barrier(p.count, base + 3ull * G);
  tstamp(7);

  // ---------------- D: fc2 + bias + residual ----------------
  rows_g2s<8>(sA, ldf, p.mid, M, F);
  __syncthreads();
  tstamp(14);
  mbar_wait(&wbar[2], 0);
  tstamp(15);
  proj_mma(sA, sW2, ldf, M, F, h0, h1, sRed, [&](int m, int n, float v) {
    const float x = sR[m * p.nh + (n - h0)] + (v + __half2float(sB2[n - h0]));
    p.hres[static_cast<long long>(m) * H + n] = x;
  });
  tstamp(8);
  grid_barrier(p.count, base + 4ull * G);
  pdl_trigger();  // every CTA of this grid is resident and past its last grid barrier

  // ---------------- E: LayerNorm of the new residual (every CTA), the next layer's q, k, v ----------------
  if (p.lnx_out == nullptr) return;
  for (int r = warp; r < M; r += kTailWarps)
    warp_layernorm_row(p.hres + static_cast<long long>(r) * H, H, sGx, sBx, p.eps, sA + r * ldh);
  __syncthreads();
  if (c == 0) {  // the normalised rows: the next layer's X slot (or the final LN's output), and its host store
    const int per_row = H >> 3;
    for (int i = threadIdx.x; i < M * per_row; i += kTailThreads) {
      const int m = i / per_row;
      const uint4 v = reinterpret_cast<const uint4*>(sA + m * ldh)[i - m * per_row];
      reinterpret_cast<uint4*>(p.lnx_out + static_cast<long long>(m) * p.lnx_ld)[i - m * per_row] = v;
      if (p.x_store != nullptr) reinterpret_cast<uint4*>(p.x_store + static_cast<long long>(m) * H)[i - m * per_row] = v;
    }
  }
  if (q1 > q0) {
    mbar_wait(&wbar[3], 0);
    // q, k, v of the new token: + bias, fp16 (the swap-AB epilogue's arithmetic) into a staging tile,
    // then 16-byte stores of whole 8-column units: q, the device page and its host copy
    __half* sQ = reinterpret_cast<__half*>(sRed);  // [M][nq]
    proj_mma_kseq(sA, sWq, ldh, M, H, q0, q1, [&](int m, int n, float v) {
      sQ[m * nq + (n - q0)] = __float2half_rn(v + __half2float(sBq[n - q0]));
    });
    __syncthreads();
    const int units = (q1 - q0) >> 3;
    for (int i = threadIdx.x; i < M * units; i += kTailThreads) {
      const int m = i / units, u = i - m * units;
      const int n = q0 + 8 * u, seg = n / H, col = n - seg * H;
      const uint4 v = *reinterpret_cast<const uint4*>(sQ + m * nq + 8 * u);
      const long long off = static_cast<long long>(m) * H + col;
      if (seg == 0) {
        *reinterpret_cast<uint4*>(p.q_out + off) = v;
      } else {
        *reinterpret_cast<uint4*>(p.page_out + static_cast<long long>(seg - 1) * M * H + off) = v;
        if (p.page_store != nullptr)
          *reinterpret_cast<uint4*>(p.page_store + static_cast<long long>(seg - 1) * M * H + off) = v;
      }
    }
  }
  tstamp(9);
}

unsigned long long* tail_count_for(int dev, cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, unsigned long long*> blocks;
  std::lock_guard<std::mutex> lock(mu);
  auto it = blocks.find({dev, stream});
  if (it != blocks.end()) return it->second;
  unsigned long long* p = nullptr;
  if (cudaMalloc(&p, kTailSyncWords * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemsetAsync(p, 0, kTailSyncWords * sizeof(unsigned long long), stream) != cudaSuccess) {
    set_error("layer tail: arrival counter allocation failed");
    return nullptr;
  }
  blocks[{dev, stream}] = p;
  return p;
}

template <int D>
int launch_tail(const TailParams& p, int grid, size_t smem, cudaStream_t stream) {
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(layer_tail_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kTailSmemBudget));
    attr_done[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTailThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, layer_tail_kernel<D>, p);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    set_error("decode_layer_tail: launch failed: %s", cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return check_launch("decode_layer_tail");
}

// (sequence, head) splits: the items cover the grid about once, >= 16 positions per split
int tail_splits(int pairs, int seq_len, int G) {
  int splits = G / pairs;
  if (splits < 1) splits = 1;
  const int max_by_len = (seq_len + 15) / 16;
  if (splits > max_by_len) splits = max_by_len;
  if (splits < 1) splits = 1;
  const int chunk = (seq_len + splits - 1) / splits;
  return (seq_len + chunk - 1) / chunk;
}

// dynamic shared memory of one launch; the item count is bounded by the grid (pairs * splits <= G
// unless pairs > G, then pairs)
size_t tail_smem_bytes(int batch, int hidden, int heads, int ffn, int G) {
  const int D = hidden / heads;
  const int nh = (hidden + G - 1) / G, nf = (ffn + G - 1) / G;
  const int pairs = batch * heads;
  const int items = pairs >= G ? pairs : (G / pairs) * pairs;
  return tail_smem(batch, hidden, ffn, nh, nf, tail_nq(hidden, G), items, D).total;
}

// CTAs of the tail grid: every SM by default; KVPR_TAIL_CTAS=n leaves SMs to a concurrent K1 (A/B)
int tail_grid(int dev) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("KVPR_TAIL_CTAS");
    env = (e != nullptr && atoi(e) > 0) ? atoi(e) : 0;
  }
  const int sms = sm_count(dev);
  return env > 0 && env < sms ? env : sms;
}

}  // namespace

bool layer_tail_supported(int batch, int hidden, int heads, int ffn) {
  if (heads <= 0 || hidden % heads != 0) return false;
  const int d = hidden / heads;
  if (!(batch >= 1 && batch <= 8 && (d == 64 || d == 128) && hidden % 16 == 0 && ffn % 16 == 0 && hidden <= 1024))
    return false;
  int dev = 0;
  cudaGetDevice(&dev);
  const int G = tail_grid(dev);
  if ((hidden + G - 1) / G > 16 * kTailMaxTiles || (ffn + G - 1) / G > 16 * kTailMaxTiles ||
      tail_nq(hidden, G) > 16 * kTailWarps)
    return false;
  return tail_smem_bytes(batch, hidden, heads, ffn, G) <= kTailSmemBudget;
}

int layer_tail(const kvpr_layer_tail_desc& d, cudaStream_t stream) {
  if (!layer_tail_supported(d.batch, d.hidden, d.heads, d.ffn) || d.head_dim * d.heads != d.hidden) {
    set_error("decode_layer_tail: needs 1 <= batch <= 8, head_dim = hidden / heads in {64, 128}, hidden <= 1024, "
              "hidden and ffn multiples of 16, and the per-CTA weight rows in shared memory "
              "(batch=%d hidden=%d heads=%d head_dim=%d ffn=%d)",
              d.batch, d.hidden, d.heads, d.head_dim, d.ffn);
    return KVPR_EINVAL;
  }
  if (d.seq_len <= 0) {
    set_error("cannot attend over an empty cache (seq_len=%d)", d.seq_len);
    return KVPR_EINVAL;
  }
  const void* ptrs16[] = {d.q, d.kv_pages, d.attn, d.wo, d.w1, d.w2, d.mid, d.hres, d.ws};
  for (const void* ptr : ptrs16) {
    if (ptr == nullptr || (reinterpret_cast<uintptr_t>(ptr) & 15)) {
      set_error("decode_layer_tail: q, kv_pages, attn, w_o, w_1, w_2, mid, hres and ws must be non-null and 16-byte aligned");
      return KVPR_EINVAL;
    }
  }
  if (d.bo == nullptr || d.b1 == nullptr || d.b2 == nullptr || d.ln2_g == nullptr || d.ln2_b == nullptr ||
      ((reinterpret_cast<uintptr_t>(d.ln2_g) | reinterpret_cast<uintptr_t>(d.ln2_b)) & 15)) {
    set_error("decode_layer_tail: biases and 16-byte aligned LN2 parameters are required");
    return KVPR_EINVAL;
  }
  if (d.lnx_out != nullptr && (d.lnx_g == nullptr || d.lnx_b == nullptr || d.lnx_ld < d.hidden || d.lnx_ld % 4 != 0 ||
                               (reinterpret_cast<uintptr_t>(d.lnx_out) & 7) ||
                               ((reinterpret_cast<uintptr_t>(d.lnx_g) | reinterpret_cast<uintptr_t>(d.lnx_b)) & 15))) {
    set_error("decode_layer_tail: the optional output LayerNorm needs gamma, beta and an 8-byte aligned output with ld >= hidden, ld %% 4 == 0");
    return KVPR_EINVAL;
  }
  if (d.kv_host != nullptr && (d.host_lo < 0 || d.host_hi > d.seq_len || (reinterpret_cast<uintptr_t>(d.kv_host) & 15))) {
    set_error("decode_layer_tail: host KV range [%d, %d) outside [0, %d) or kv_host not 16-byte aligned", d.host_lo,
              d.host_hi, d.seq_len);
    return KVPR_EINVAL;
  }
  if ((d.x_store_next != nullptr && (d.lnx_out == nullptr || (reinterpret_cast<uintptr_t>(d.x_store_next) & 15))) ||
      (d.page_store_next != nullptr && d.wqkv_next == nullptr)) {
    set_error("decode_layer_tail: x_store_next needs the output LayerNorm (16-byte aligned), page_store_next the "
              "next layer's q/k/v");
    return KVPR_EINVAL;
  }
  if (d.wqkv_next != nullptr &&
      (d.lnx_out == nullptr || d.bqkv_next == nullptr || d.q_next == nullptr || d.page_next == nullptr ||
       ((reinterpret_cast<uintptr_t>(d.wqkv_next) | reinterpret_cast<uintptr_t>(d.q_next) |
         reinterpret_cast<uintptr_t>(d.page_next)) & 15))) {
    set_error("decode_layer_tail: the next layer's q/k/v needs the output LayerNorm, its bias, and 16-byte aligned "
              "w_qkv, q and page pointers");
    return KVPR_EINVAL;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  const int G = tail_grid(dev);
  const int D = d.head_dim;
  const int pairs = d.batch * d.heads;
  const int splits = tail_splits(pairs, d.seq_len, G);
  const int chunk = (d.seq_len + splits - 1) / splits;
  const size_t part_bytes = static_cast<size_t>(pairs) * splits * (D + 4) * sizeof(float);
  if (part_bytes > d.ws_bytes) {
    set_error("decode_layer_tail: workspace of %zu B below the %zu B of attention partials", d.ws_bytes, part_bytes);
    return KVPR_EINVAL;
  }
  unsigned long long* count = tail_count_for(dev, stream);
  if (count == nullptr) return KVPR_ECUDA;
  TailParams p;
  p.M = d.batch;
  p.H = d.hidden;
  p.heads = d.heads;
  p.F = d.ffn;
  p.S = d.seq_len;
  p.qscale = d.scale * 1.4426950408889634f;
  p.eps = d.eps;
  p.q = static_cast<const __half*>(d.q);
  p.kv = static_cast<const __half*>(d.kv_pages);
  p.attn = static_cast<__half*>(d.attn);
  p.wo = static_cast<const __half*>(d.wo);
  p.bo = static_cast<const __half*>(d.bo);
  p.hres = d.hres;
  p.ln2_g = static_cast<const __half*>(d.ln2_g);
  p.ln2_b = static_cast<const __half*>(d.ln2_b);
  p.w1 = static_cast<const __half*>(d.w1);
  p.b1 = static_cast<const __half*>(d.b1);
  p.mid = static_cast<__half*>(d.mid);
  p.w2 = static_cast<const __half*>(d.w2);
  p.b2 = static_cast<const __half*>(d.b2);
  p.lnx_g = static_cast<const __half*>(d.lnx_g);
  p.lnx_b = static_cast<const __half*>(d.lnx_b);
  p.lnx_out = static_cast<__half*>(d.lnx_out);
  p.lnx_ld = d.lnx_ld;
  p.wq = static_cast<const __half*>(d.wqkv_next);
  p.bq = static_cast<const __half*>(d.bqkv_next);
  p.q_out = static_cast<__half*>(d.q_next);
  p.page_out = static_cast<__half*>(d.page_next);
  p.kv_alt = static_cast<const __half*>(d.kv_host);
  p.alt_lo = d.host_lo;
  p.alt_hi = d.host_hi;
  p.x_store = static_cast<__half*>(d.x_store_next);
  p.page_store = static_cast<__half*>(d.page_store_next);
  p.part = static_cast<float*>(d.ws);
  p.count = count;
  p.splits = splits;
  p.chunk = chunk;
  p.nh = (d.hidden + G - 1) / G;
  p.nf = (d.ffn + G - 1) / G;
  // the host tail of each attention item pulled into shared memory at entry when it is small (the
  // usual case: l close to s'), else read in place
  p.alt_npos = 0;
  if (d.kv_host != nullptr && d.host_hi > d.host_lo) {
    const int npos = d.host_hi - d.host_lo < chunk ? d.host_hi - d.host_lo : chunk;
    const int per_cta = (pairs * splits + G - 1) / G;
    const uint32_t hb = static_cast<uint32_t>(per_cta) * npos * 2 * D * 2;
    if (hb <= 16 * 1024 &&
        tail_smem(d.batch, d.hidden, d.ffn, p.nh, p.nf, tail_nq(d.hidden, G), pairs * splits, D, hb).total <=
            kTailSmemBudget)
      p.alt_npos = npos;
  }
  const size_t smem = tail_smem(d.batch, d.hidden, d.ffn, p.nh, p.nf, tail_nq(d.hidden, G), pairs * splits, D,
                                static_cast<uint32_t>(((pairs * splits + G - 1) / G) * p.alt_npos * 2 * D * 2)).total;
  if (D == 128) return launch_tail<128>(p, G, smem, stream);
  return launch_tail<64>(p, G, smem, stream);
}

// Diagnostic (tests/test_layer_tail_gpu.py): out[m][n] = sum_k a[m][k] w[n][k] on the warp tensor
// cores with the k order of the tcgen05 kernels (16-wide steps, ascending, one accumulator per
// element) -- whether mma.sync reproduces tcgen05.mma's bits.  One warp per 16 columns; M <= 8.
__global__ void mma_linear_probe_kernel(const __half* a, const __half* w, float* out, int M, int N, int K) {
  const int lane = threadIdx.x & 31;
  const int n0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 16;
  if (n0 >= N) return;
  const int g = lane >> 2, q = lane & 3;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < K; k0 += 16) {
    // fragments straight from global (row-major A tile = weights rows n0.., B = activation rows)
    auto wv = [&](int r, int k) -> uint32_t {
      const int n = n0 + r;
      if (n >= N) return 0u;
      return *reinterpret_cast<const uint32_t*>(w + static_cast<long long>(n) * K + k);
    };
    auto av = [&](int m, int k) -> uint32_t {
      if (m >= M) return 0u;
      return *reinterpret_cast<const uint32_t*>(a + static_cast<long long>(m) * K + k);
    };
    uint32_t fa[4] = {wv(g, k0 + 2 * q), wv(g + 8, k0 + 2 * q), wv(g, k0 + 8 + 2 * q), wv(g + 8, k0 + 8 + 2 * q)};
    uint32_t fb[2] = {av(g, k0 + 2 * q), av(g, k0 + 8 + 2 * q)};
    mma_16816(acc, fa, fb);
  }
  const int m0 = 2 * q;
  if (n0 + g < N) {
    if (m0 < M) out[static_cast<long long>(m0) * N + n0 + g] = acc[0];
    if (m0 + 1 < M) out[static_cast<long long>(m0 + 1) * N + n0 + g] = acc[1];
  }
  if (n0 + g + 8 < N) {
    if (m0 < M) out[static_cast<long long>(m0) * N + n0 + g + 8] = acc[2];
    if (m0 + 1 < M) out[static_cast<long long>(m0 + 1) * N + n0 + g + 8] = acc[3];
  }
}

}  // namespace kvpr

extern "C" int kvpr_debug_mma_linear(const void* a, const void* w, float* out, int M, int N, int K, void* stream) {
  if (M < 1 || M > 8 || N < 1 || K % 16 != 0) return KVPR_EINVAL;
  const int warps = 4, grid = (N + 16 * warps - 1) / (16 * warps);
  kvpr::mma_linear_probe_kernel<<<grid, 32 * warps, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __half*>(a), static_cast<const __half*>(w), out, M, N, K);
  return cudaGetLastError() == cudaSuccess ? KVPR_OK : KVPR_ECUDA;
}

extern "C" int kvpr_debug_tail_trace(void* buf) {  // tools/tail_bench.py: 24 u64 stamps per CTA, NULL = off
  return cudaMemcpyToSymbol(kvpr::g_tail_trace, &buf, sizeof(buf)) == cudaSuccess ? KVPR_OK : KVPR_ECUDA;
}
