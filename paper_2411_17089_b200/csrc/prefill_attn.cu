// Causal prefill attention on the 5th-generation tensor cores (flash schedule, tcgen05.mma with the
// S and O accumulators in TMEM).
//
// Reference semantics: the prompt pass that produces the per-layer host stores X and KV; per
// (sequence, head) softmax(Q K^T / sqrt(d) + causal mask) V, the same attention
// numerics.decode_attention (numerics.py:166-191) applies per position.  Off the timed decode path
// (the reference prices it nowhere: pipesim models decode layers only), but it gates long-prompt
// runs (config 5, prompt 8192): the CUDA-core kernel of round 1 spent 36 ms per OPT-6.7B layer at
// b32 s1024, a warp-MMA (mma.sync) flash kernel 1.27 ms, this one 0.67 ms
// (profiles/r02_prefill_bench.jsonl).
//
// Layout (runtime.py prefill): q rows [pos][b][hidden]; KV pages [pos][2][b][hidden] -- one
// (sequence, head) row of K or V is head_dim contiguous halves, rows of consecutive positions are
// b*hidden (q) or 2*b*hidden (K, V) halves apart: 3-D TMA maps (h, b or 2b, pos) cut 64-column x
// 128-position boxes straight out of them.  The output goes to [pos][b][hidden] like q.
//
// One CTA per (128-query tile, sequence, head), heaviest (last) query tiles first.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {
namespace {

// Warp roles (256 threads): w0 = TMA producer, w1 = MMA issuer (one elected lane), w2 = TMEM
// allocator, w4..w7 = softmax / O correction / epilogue with thread t <-> TMEM lane t <-> query row
// q0 + t (a whole S row per thread: max and sum need no shuffles).  Per key tile j:
//   MMA    S_j = Q K_j^T -> TMEM S[j % 2]                      (commit sfull[j % 2])
//          after P_{j-1} is in smem: O += P_{j-1} V_{j-1}      (commit pvdone, kvempty)
//   softmax  S_j -> registers, scale, causal mask, row max m', p = exp2(s - m'), row sum;
//          after pvdone(j-1): O *= exp2(m - m') in TMEM if the max moved, P_j -> smem (fp16,
//          K-major SW128) -> arrive pfull
// so S_{j+1} runs on the tensor core while the softmax of S_j runs, and P V of tile j while the
// softmax of tile j+1 computes its row statistics.  Q, K, V by TMA (3-D maps over the [pos][b][h]
// and [pos][2][b][h] layouts, 128-row boxes, zero fill past seq_len); V is read MN-major (the
// instruction's B-transpose bit), P V's A operand is P in shared memory.
namespace tc {

constexpr int kRows = 128;  // queries per CTA and keys per tile

template <int D>
struct Cfg {
  static constexpr uint32_t kBox = kRows * 64 * 2;      // one 64-column box: 16 KB
  static constexpr uint32_t kTile = kRows * D * 2;      // Q, K or V tile
  static constexpr uint32_t kQ = 0, kK = kTile, kV = 3 * kTile, kP = 5 * kTile;
  static constexpr uint32_t kBar = kP + kRows * kRows * 2;
  static constexpr uint32_t kSmem = kBar + 256 + 1024;  // barriers, 1024-B alignment slack
  static constexpr uint32_t kO = 2 * kRows;              // TMEM column of O (S[0] at 0, S[1] at 128)
};

// bounded wait: a schedule bug traps (a launch error) instead of hanging the GPU; `code` / `j` name the
// wait in a debugger
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity, int code = 0, int j = 0) {
  const uint32_t a = smem_u32(bar);
  for (uint32_t i = 0; !mbar_try_wait(a, parity); ++i)
    if (i == (1u << 30)) {
      (void)code;
      (void)j;
      __trap();
    }
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// MN-major operand with the 128-byte swizzle: 64-element (128 B) rows along N, 8-row atoms along K
// 1024 B apart (SBO), consecutive 64-element N blocks `lbo` bytes apart (LBO)
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

template <int D>
__global__ void __launch_bounds__(256, 1) prefill_tc_kernel(const __grid_constant__ CUtensorMap tq,
                                                           const __grid_constant__ CUtensorMap tkv,
                                                           __half* __restrict__ out, int batch, int heads,
                                                           int seq_len, float qscale) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t base = smem_u32(sm);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::kBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* v_full = bars + 3;   // [2]
  uint64_t* kv_empty = bars + 5; // [2]
  uint64_t* s_full = bars + 7;   // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* pv_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int qt = gridDim.x - 1 - blockIdx.x;  // long (late) query tiles first
  const int b = blockIdx.y / heads, hd = blockIdx.y % heads;
  const int q0 = qt * kRows, ntiles = qt + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tkv);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(bars + i, 1);
    mbar_init(p_full, 128);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      mbar_arrive_expect_tx(q_full, C::kTile);
      for (int c = 0; c < D / 64; ++c) tma_load_3d(base + C::kQ + c * C::kBox, &tq, q_full, hd * D + c * 64, b, q0);
      for (int j = 0; j < ntiles; ++j) {
        const int buf = j & 1;
        if (j >= 2) wait_bar(&kv_empty[buf], ((j - 2) >> 1) & 1, 1, j);
        mbar_arrive_expect_tx(&k_full[buf], C::kTile);
        for (int c = 0; c < D / 64; ++c)
          tma_load_3d(base + C::kK + buf * C::kTile + c * C::kBox, &tkv, &k_full[buf], hd * D + c * 64, b, j * kRows);
        mbar_arrive_expect_tx(&v_full[buf], C::kTile);
        for (int c = 0; c < D / 64; ++c)
          tma_load_3d(base + C::kV + buf * C::kTile + c * C::kBox, &tkv, &v_full[buf], hd * D + c * 64, batch + b,
                      j * kRows);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_s = umma_idesc_f16_f32(kRows, kRows);
      constexpr uint32_t idesc_o = umma_idesc_f16_f32(kRows, D) | (1u << 16);  // B (V) MN-major
      wait_bar(q_full, 0, 2);
      tc_fence_after();
      for (int j = 0; j <= ntiles; ++j) {
        if (j < ntiles) {  // S_j = Q K_j^T (its S buffer was released with P_{j-2})
          const int buf = j & 1;
          wait_bar(&k_full[buf], (j >> 1) & 1, 3, j);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16(tmem + buf * kRows, umma_desc_k_sw128(base + C::kQ + c * C::kBox + k * 32),
                       umma_desc_k_sw128(base + C::kK + buf * C::kTile + c * C::kBox + k * 32), idesc_s,
                       (c | k) != 0);
          umma_commit(&s_full[buf]);
        }
        if (j >= 1) {  // O += P_{j-1} V_{j-1}
          const int i = j - 1, ib = i & 1;
          wait_bar(p_full, i & 1, 4, i);
          wait_bar(&v_full[ib], (i >> 1) & 1, 5, i);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kRows / 16; ++kk)
            umma_f16(tmem + C::kO, umma_desc_k_sw128(base + C::kP + (kk >> 2) * C::kBox + (kk & 3) * 32),
                     desc_mn_sw128(base + C::kV + ib * C::kTile + kk * 2048, C::kBox), idesc_o, (i | kk) != 0);
          umma_commit(pv_done);
          umma_commit(&kv_empty[ib]);
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- softmax, O correction, epilogue ----------------
    const int t = threadIdx.x - 128;
    const uint32_t lanes = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    const int row = q0 + t;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int buf = j & 1;
      wait_bar(&s_full[buf], (j >> 1) & 1, 6, j);
      tc_fence_after();
      float s[kRows];
#pragma unroll
      for (int cc = 0; cc < kRows / 32; ++cc) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + lanes + buf * kRows + cc * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[cc * 32 + i] = __uint_as_float(r[i]) * qscale;
      }
      if (j == ntiles - 1) {  // diagonal tile: keys past the query (and past seq_len) masked
#pragma unroll
        for (int c = 0; c < kRows; ++c)
          if (j * kRows + c > row) s[c] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kRows; ++c) mx = fmaxf(mx, s[c]);
      // lazy rescaling: keep the running max unless this tile exceeds it by more than 2^8 (P <= 256
      // stays exact enough in fp16 and O / l absorb the common factor), so most tiles after the first
      // skip the O correction; the first tile always sets it (finite: key j*128 <= row on every tile)
      mx = (mx > m + 8.f) ? mx : m;
      const float alpha = exp2f(m - mx);
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < kRows; ++c) {
        s[c] = exp2f(s[c] - mx);
        sum += s[c];
      }
      l = l * alpha + sum;
      m = mx;
      if (j >= 1) {  // P V of the previous tile is done: O and the P buffer are ours
        wait_bar(pv_done, (j - 1) & 1, 7, j);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {  // warp-uniform: tcgen05.ld/st are .sync.aligned
#pragma unroll 1
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem + lanes + C::kO + cc * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st_x32(tmem + lanes + C::kO + cc * 32, r);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
      // P row t -> shared memory, K-major with the 128-byte swizzle (16-byte unit u of row t at u ^ (t & 7))
#pragma unroll
      for (int u = 0; u < kRows / 8; ++u) {
        uint4 v;
        v.x = pack_half2(s[u * 8 + 0], s[u * 8 + 1]);
        v.y = pack_half2(s[u * 8 + 2], s[u * 8 + 3]);
        v.z = pack_half2(s[u * 8 + 4], s[u * 8 + 5]);
        v.w = pack_half2(s[u * 8 + 6], s[u * 8 + 7]);
        const uint32_t addr = base + C::kP + (u >> 3) * C::kBox + t * 128 + (((u & 7) ^ (t & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy P writes -> tcgen05 reads
      tc_fence_before();
      mbar_arrive(p_full);
    }
    wait_bar(pv_done, (ntiles - 1) & 1, 8, ntiles);
    tc_fence_after();
    const float inv = 1.f / l;
    __half* o = out + (static_cast<long long>(row) * batch + b) * heads * D + hd * D;
#pragma unroll 1
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + lanes + C::kO + cc * 32, r);
      tmem_ld_wait();
      if (row < seq_len) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 v;
          v.x = pack_half2(__uint_as_float(r[u * 8 + 0]) * inv, __uint_as_float(r[u * 8 + 1]) * inv);
          v.y = pack_half2(__uint_as_float(r[u * 8 + 2]) * inv, __uint_as_float(r[u * 8 + 3]) * inv);
          v.z = pack_half2(__uint_as_float(r[u * 8 + 4]) * inv, __uint_as_float(r[u * 8 + 5]) * inv);
          v.w = pack_half2(__uint_as_float(r[u * 8 + 6]) * inv, __uint_as_float(r[u * 8 + 7]) * inv);
          reinterpret_cast<uint4*>(o + cc * 32)[u] = v;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace tc

template <int D>
int launch_prefill_tc(const __half* q, const __half* kv, __half* out, int batch, int heads, int seq_len,
                      float qscale, cudaStream_t stream) {
  using C = tc::Cfg<D>;
  const uint64_t hidden = static_cast<uint64_t>(heads) * D;
  CUtensorMap tq, tkv;
  // q [pos][b][h] and the pages [pos][2][b][h] as (h, b or 2b, pos); 64-column x 128-position boxes
  const uint64_t qd[3] = {hidden, static_cast<uint64_t>(batch), static_cast<uint64_t>(seq_len)};
  const uint64_t qs[2] = {hidden * 2, hidden * 2 * batch};
  const uint64_t kd[3] = {hidden, 2ull * batch, static_cast<uint64_t>(seq_len)};
  const uint64_t ks[2] = {hidden * 2, hidden * 4 * batch};
  const uint32_t box[3] = {64, 1, static_cast<uint32_t>(tc::kRows)};
  int rc = make_tmap_nd(&tq, q, 3, qd, qs, box);
  if (rc == KVPR_OK) rc = make_tmap_nd(&tkv, kv, 3, kd, ks, box);
  if (rc != KVPR_OK) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_done[64] = {0};
  if (dev >= 64 || !attr_done[dev]) {
    cudaFuncSetAttribute(tc::prefill_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    if (dev < 64) attr_done[dev] = 1;
  }
  dim3 grid((seq_len + tc::kRows - 1) / tc::kRows, batch * heads);
  tc::prefill_tc_kernel<D><<<grid, 256, C::kSmem, stream>>>(tq, tkv, out, batch, heads, seq_len, qscale);
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
  if (head_dim == 128) return launch_prefill_tc<128>(q, kv, out, batch, heads, seq_len, qscale, stream);
  return launch_prefill_tc<64>(q, kv, out, batch, heads, seq_len, qscale, stream);
}

}  // namespace kvpr
