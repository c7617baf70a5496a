// Causal prefill attention on the tensor cores (flash-attention schedule, mma.sync m16n8k16).
//
// Reference semantics: the prompt pass that produces the per-layer host stores X and KV; per
// (sequence, head) softmax(Q K^T / sqrt(d) + causal mask) V, the same attention
// numerics.decode_attention (numerics.py:166-191) applies per position.  Off the timed decode path
// (the reference prices it nowhere: pipesim models decode layers only), but it gates long-prompt
// runs (config 5, prompt 8192): the CUDA-core version this replaces spent 36 ms per OPT-6.7B layer
// at b32 s1024 (profiles/r01_launches_summary.txt).
//
// Layout (runtime.py prefill): q rows [pos][b][hidden]; KV pages [pos][2][b][hidden] -- one
// (sequence, head) row of K or V is head_dim contiguous halves, rows of consecutive positions are
// 2*b*hidden halves apart.  The output goes to [pos][b][hidden] like q.
//
// Tiling: one CTA per (64-query tile, sequence, head), heaviest (last) query tiles first; 4 warps,
// warp w owns query rows 16w..16w+15.  Per 64-key tile: S = Q K^T (Q fragments held in registers for
// the whole CTA), scale + causal mask in fp32, online softmax in the exp2 domain (each thread owns
// two query rows, max / sum over the 4-lane quad), P rounded to fp16 straight from the S
// accumulators into A fragments, O += P V with V fragments from ldmatrix.trans.  K/V tiles are
// double-buffered with cp.async (16 B, zero-fill past seq_len); shared rows are XOR-swizzled in
// 16-byte chunks (chunk ^ (row & 7)) so every ldmatrix phase hits 8 distinct bank groups.

#include <math.h>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {
namespace {

constexpr int kBM = 64;  // query rows per CTA
constexpr int kBN = 64;  // keys per tile

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// byte offset of 16-byte chunk c of row r in a swizzled [rows][D] half tile
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)(r * (D * 2) + ((c ^ (r & 7)) << 4));
}

// rows [p0, p0 + 64) of a [pos]-strided operand into a swizzled tile; rows >= seq_len read as zero
template <int D>
__device__ __forceinline__ void load_tile(uint32_t dst, const __half* base, long long stride, int p0, int seq_len) {
  constexpr int CPR = D / 8;  // 16-byte chunks per row
#pragma unroll
  for (int i = threadIdx.x; i < kBN * CPR; i += 128) {
    const int r = i / CPR, c = i % CPR;
    const bool ok = p0 + r < seq_len;
    cp_async16(dst + swz<D>(r, c), base + (ok ? (long long)(p0 + r) * stride : 0) + c * 8, ok);
  }
}

template <int D>
__global__ void __launch_bounds__(128) prefill_fa_kernel(const __half* __restrict__ q, const __half* __restrict__ kv,
                                                         __half* __restrict__ out, int batch, int heads, int seq_len,
                                                         float qscale) {
  constexpr int KS = D / 16;  // k-steps of S = Q K^T
  constexpr int DB = D / 8;   // 8-wide output column blocks
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + kBM * D * 2;
  const uint32_t sV0 = sK0 + 2 * kBN * D * 2;
  constexpr uint32_t kTile = kBN * D * 2;

  const int qt = gridDim.x - 1 - blockIdx.x;  // long (late) query tiles first
  const int bh = blockIdx.y;
  const int b = bh / heads, hd = bh % heads;
  const long long hidden = (long long)heads * D;
  const long long qstride = (long long)batch * hidden;
  const long long kstride = 2 * qstride;
  const __half* qb = q + b * hidden + hd * D;
  const __half* kb = kv + b * hidden + hd * D;
  const __half* vb = kb + qstride;
  const int q0 = qt * kBM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  load_tile<D>(sQ, qb, qstride, q0, seq_len);
  load_tile<D>(sK0, kb, kstride, 0, seq_len);
  load_tile<D>(sV0, vb, kstride, 0, seq_len);
  cp_async_commit();

  uint32_t qf[KS][4];
  float o[DB][4];
#pragma unroll
  for (int i = 0; i < DB; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int row0 = q0 + warp * 16 + g;  // this thread's two query rows: row0, row0 + 8

  for (int kt = 0; kt <= qt; ++kt) {
    const int buf = kt & 1;
    if (kt < qt) {  // prefetch the next K/V tile into the other buffer
      load_tile<D>(sK0 + (buf ^ 1) * kTile, kb, kstride, (kt + 1) * kBN, seq_len);
      load_tile<D>(sV0 + (buf ^ 1) * kTile, vb, kstride, (kt + 1) * kBN, seq_len);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) ldsm_x4(sQ + swz<D>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), qf[kk]);
    }
    const uint32_t sK = sK0 + buf * kTile, sV = sV0 + buf * kTile;

    // S = Q K^T: 8 column blocks of 8 keys
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int nb2 = 0; nb2 < 4; ++nb2) {
      const int kr = nb2 * 16 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        uint32_t r[4];
        ldsm_x4(sK + swz<D>(kr, kk * 2 + ((lane >> 3) & 1)), r);
        mma16816(s[2 * nb2], qf[kk], r[0], r[1]);
        mma16816(s[2 * nb2 + 1], qf[kk], r[2], r[3]);
      }
    }
    // scale into the exp2 domain; causal mask on the diagonal tile (also masks keys >= seq_len there)
    const bool diag = kt == qt;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const int key = kt * kBN + nb * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[nb][e] * qscale;
        if (diag && key + (e & 1) > row0 + ((e >> 1) << 3)) v = -INFINITY;
        s[nb][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(s[nb][0], s[nb][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nb][2], s[nb][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);  // finite: every row sees key 0 in tile 0
    const float a0 = exp2f(m0 - n0), a1 = exp2f(m1 - n1);
    m0 = n0;
    m1 = n1;
    float r0 = 0.f, r1 = 0.f;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      s[nb][0] = exp2f(s[nb][0] - n0);
      s[nb][1] = exp2f(s[nb][1] - n0);
      s[nb][2] = exp2f(s[nb][2] - n1);
      s[nb][3] = exp2f(s[nb][3] - n1);
      r0 += s[nb][0] + s[nb][1];
      r1 += s[nb][2] + s[nb][3];
    }
    l0 = l0 * a0 + r0;
    l1 = l1 * a1 + r1;
#pragma unroll
    for (int i = 0; i < DB; ++i) {
      o[i][0] *= a0;
      o[i][1] *= a0;
      o[i][2] *= a1;
      o[i][3] *= a1;
    }
    // O += P V: P's fp16 A fragments come straight from the S accumulators (16 keys per k-step)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_half2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_half2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_half2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_half2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
      const int vr = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
      for (int db2 = 0; db2 < DB / 2; ++db2) {
        uint32_t r[4];
        ldsm_x4_t(sV + swz<D>(vr, db2 * 2 + (lane >> 4)), r);
        mma16816(o[2 * db2], pa, r[0], r[1]);
        mma16816(o[2 * db2 + 1], pa, r[2], r[3]);
      }
    }
    __syncthreads();  // the buffer this tile used is refilled by the next iteration's prefetch
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  __half* ob = out + b * hidden + hd * D + 2 * t;
#pragma unroll
  for (int db = 0; db < DB; ++db) {
    if (row0 < seq_len)
      *reinterpret_cast<uint32_t*>(ob + (long long)row0 * qstride + db * 8) = pack_half2(o[db][0] * i0, o[db][1] * i0);
    if (row0 + 8 < seq_len)
      *reinterpret_cast<uint32_t*>(ob + (long long)(row0 + 8) * qstride + db * 8) =
          pack_half2(o[db][2] * i1, o[db][3] * i1);
  }
}

template <int D>
int launch_prefill(const __half* q, const __half* kv, __half* out, int batch, int heads, int seq_len, float qscale,
                   cudaStream_t stream) {
  constexpr size_t smem = (size_t)(kBM + 4 * kBN) * D * 2;
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_done[64] = {0};  // the attribute is per device
  if (dev >= 64 || !attr_done[dev]) {
    cudaFuncSetAttribute(prefill_fa_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev < 64) attr_done[dev] = 1;
  }
  dim3 grid((seq_len + kBM - 1) / kBM, batch * heads);
  prefill_fa_kernel<D><<<grid, 128, smem, stream>>>(q, kv, out, batch, heads, seq_len, qscale);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return check_launch("prefill_attention");
}

}  // namespace

int prefill_attention(const __half* q, const __half* kv, __half* out, int batch, int heads, int head_dim, int seq_len,
                      float scale, cudaStream_t stream) {
  if (seq_len <= 0 || batch <= 0 || heads <= 0 || (head_dim != 64 && head_dim != 128) ||
      (long long)batch * heads > 65535) {
    set_error("prefill_attention: bad shape seq=%d batch=%d heads=%d head_dim=%d", seq_len, batch, heads, head_dim);
    return KVPR_EINVAL;
  }
  const float qscale = scale * 1.4426950408889634f;
  if (head_dim == 128) return launch_prefill<128>(q, kv, out, batch, heads, seq_len, qscale, stream);
  return launch_prefill<64>(q, kv, out, batch, heads, seq_len, qscale, stream);
}

}  // namespace kvpr
