// Causal prefill attention on the 5th-generation tensor cores (flash schedule, tcgen05.mma with the
// S and O accumulators in TMEM).
//
// Reference semantics: the prompt pass that produces the per-layer host stores X and KV; per
// (sequence, head) softmax(Q K^T / sqrt(d) + causal mask) V, the same attention
// numerics.decode_attention (numerics.py:166-191) applies per position.  Off the timed decode path
// (the reference prices it nowhere: pipesim models decode layers only), but it gates long-prompt
// runs (config 5, prompt 8192): the CUDA-core kernel of round 1 spent 36 ms per OPT-6.7B layer at
// b32 s1024, a warp-MMA (mma.sync) flash kernel 1.27 ms, a one-query-tile tcgen05 version 0.67 ms, this
// persistent two-tile ping-pong 0.37 ms (profiles/r02_prefill_bench.jsonl).
//
// Layout (runtime.py prefill): q rows [pos][b][hidden]; KV pages [pos][2][b][hidden] -- one
// (sequence, head) row of K or V is head_dim contiguous halves, rows of consecutive positions are
// b*hidden (q) or 2*b*hidden (K, V) halves apart: 3-D TMA maps (h, b or 2b, pos) cut 64-column x
// 128-position boxes straight out of them.  The output goes to [pos][b][hidden] like q.
//
// Persistent: one CTA per SM walks the work items (pair of 128-query tiles, sequence, head).
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {
namespace {

// Two query tiles per CTA, ping-ponged (384 threads): w0 = TMA producer of Q and K, w1 = MMA issuer
// (one elected lane; the warp allocates TMEM), w2 = TMA producer of V, w4..w7 = softmax / O correction /
// epilogue of query tile A, w8..w11 the same for tile B, thread t of a group <-> TMEM lane t <-> query
// row q0 + t (a whole S row per thread: max and sum need no shuffles).  TMEM: S_A, S_B, O_A, O_B.
// Per key tile j and tile T in {A, B}:
//   MMA      once P_T(j-1) is in smem: S_T(j) = Q_T K_j^T (commit s_full[T]),
//            O_T += P_T(j-1) V_{j-1} (commit pv_done[T]); K_j / V_{j-1} released after tile B's use
//   softmax  pass 1: S_T(j) -> row max (8 independent chains); wait pv_done[T](j-1), O_T *= exp2(m - m')
//            in TMEM if the max moved; pass 2: S_T(j) again -> p = exp2(s - m'), row sum, P_T -> smem
//            (fp16, K-major SW128) -> arrive p_full[T]
// While one group runs its softmax (MUFU / FMA latency-bound: one warp per sub-partition and group) the
// tensor core works on the other group's S and P V, so the two chains hide each other.  The pair is
// two adjacent query tiles (2p, 2p+1): tile B needs one more key tile than A, heaviest pairs first.
// Q, K, V by TMA (3-D maps over the [pos][b][h] and [pos][2][b][h] layouts, 128-row boxes, zero fill past
// seq_len); V is read MN-major (the instruction's B-transpose bit), P V's A operand is P in shared memory.
namespace tc {

constexpr int kRows = 128;  // queries per tile and keys per tile
constexpr int kKS = 2;      // K stages

template <int D>
struct Cfg {
  static constexpr int kVS = D == 64 ? 2 : 1;          // V stages (D = 128: 224 KB of the 227 KB)
  static constexpr uint32_t kBox = kRows * 64 * 2;      // one 64-column box: 16 KB
  static constexpr uint32_t kTile = kRows * D * 2;      // Q, K or V tile
  static constexpr uint32_t kP1 = kRows * kRows * 2;    // one P tile: 32 KB
  static constexpr uint32_t kQ = 0, kK = 2 * kTile, kV = kK + kKS * kTile, kP = kV + kVS * kTile;
  static constexpr uint32_t kBar = kP + 2 * kP1;
  static constexpr uint32_t kSmem = kBar + 256 + 1024;  // barriers, 1024-B alignment slack
  static constexpr uint32_t kO = 2 * kRows;              // TMEM column of O_A (S_A at 0, S_B at 128)
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

__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2, flush-to-zero (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// y = x * a + c on a pair of floats in one FFMA2 (the sm_100 paired fp32 pipe)
__device__ __forceinline__ void ffma2(float& y0, float& y1, float x0, float x1, float a, float c) {
  uint64_t x, av, cv, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(cv) : "f"(c));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(y) : "l"(x), "l"(av), "l"(cv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(y0), "=f"(y1) : "l"(y));
}

// (s0, s1) += (x0, x1) in one FADD2
__device__ __forceinline__ void fadd2(float& s0, float& s1, float x0, float x1) {
  uint64_t sv, xv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(sv) : "f"(s0), "f"(s1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(xv) : "f"(x0), "f"(x1));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(sv) : "l"(xv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(s0), "=f"(s1) : "l"(sv));
}

// the row max of a 128-key score tile held in registers: 8 independent chains of 3-input max (FMNMX3)
__device__ __forceinline__ float row_max128(const uint32_t (&r)[kRows]) {
  float mp[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) mp[i] = -INFINITY;
#pragma unroll
  for (int i = 0; i < kRows; i += 2)
    mp[(i >> 1) & 7] = fmaxf(mp[(i >> 1) & 7], fmaxf(__uint_as_float(r[i]), __uint_as_float(r[i + 1])));
  return fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])), fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
}

// p = exp2(s * scale - m') (FFMA2 + MUFU.EX2; masked scores are -inf -> 0), the row sum (FADD2), P row tt
// -> shared memory, K-major with the 128-byte swizzle (16-byte unit u of row tt at u ^ (tt & 7))
__device__ __forceinline__ float exp_store128(const uint32_t (&r)[kRows], float qscale, float mx, uint32_t p_base,
                                              int tt, uint32_t box_bytes) {
  float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int u = 0; u < kRows / 8; ++u) {
    float p[8];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      ffma2(p[i], p[i + 1], __uint_as_float(r[u * 8 + i]), __uint_as_float(r[u * 8 + i + 1]), qscale, -mx);
      p[i] = ex2_approx(p[i]);
      p[i + 1] = ex2_approx(p[i + 1]);
      fadd2(sp[i >> 1], sp[(i >> 1) + 4], p[i], p[i + 1]);
    }
    const uint32_t addr = p_base + (u >> 3) * box_bytes + tt * 128 + (((u & 7) ^ (tt & 7)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pack_half2(p[0], p[1])),
                 "r"(pack_half2(p[2], p[3])), "r"(pack_half2(p[4], p[5])), "r"(pack_half2(p[6], p[7]))
                 : "memory");
  }
  return ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
}

__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
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

// One work item = (pair of query tiles, sequence, head).  Persistent: CTA c takes one item per round of
// G = gridDim.x <= #SMs items (item_of below), so one item's epilogue (O out of TMEM) overlaps the next
// item's Q / K / V loads and its first S MMAs; every barrier's phase runs on across items (per-role
// running counters), with q_empty / o_free releasing Q and O_t to the next item.
struct Item {
  int pair, b, hd, nt_a, ntk;  // nt_a / ntk: key tiles of tiles A / B (ntk >= nt_a)
};

__device__ __forceinline__ Item item_at(int w, int npair, int heads, int ktot) {
  // long (late) pairs first within each (sequence, head); the pairs of one (sequence, head) are adjacent
  // in item order so they share its K / V in L2 (pair-major order measured 3-12% slower)
  Item it;
  const int bh = w / npair;
  it.pair = npair - 1 - w % npair;
  it.b = bh / heads;
  it.hd = bh % heads;
  it.nt_a = 2 * it.pair + 1;
  it.ntk = min(2 * it.pair + 2, ktot);
  return it;
}

// the k-th item of CTA c among G: rounds of G consecutive items, walked forwards on even rounds and
// backwards on odd ones, so a CTA handed a heavy pair in one round gets a light one in the next (plain
// striding hands every CTA the same pair index whenever the pair count divides G), while the items in
// flight stay a contiguous range (the pairs of one (sequence, head) share its K / V in L2)
__device__ __forceinline__ int item_of(int k, int c, int G) { return k * G + ((k & 1) ? G - 1 - c : c); }

template <int D>
__global__ void __launch_bounds__(384, 1) prefill_tc_kernel(const __grid_constant__ CUtensorMap tq,
                                                           const __grid_constant__ CUtensorMap tkv,
                                                           __half* __restrict__ out, int batch, int heads,
                                                           int seq_len, float qscale) {
  using C = Cfg<D>;
  constexpr int VS = C::kVS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t base = smem_u32(sm);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::kBar);
  uint64_t* q_full = bars;             // [1]
  uint64_t* k_full = bars + 1;         // [kKS]
  uint64_t* k_empty = bars + 3;        // [kKS]
  uint64_t* v_full = bars + 5;         // [VS]
  uint64_t* v_empty = bars + 7;        // [VS]
  uint64_t* s_full = bars + 9;         // [2] per query tile
  uint64_t* p_full = bars + 11;        // [2]
  uint64_t* pv_done = bars + 13;       // [2]
  uint64_t* s_free = bars + 15;        // [2] S_t read into registers: TMEM S_t may be overwritten
  uint64_t* q_empty = bars + 17;       // [1] the item's last S MMAs done: Q may be reloaded
  uint64_t* o_free = bars + 18;        // [2] the item's O_t read out: the next item's first P V may overwrite it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int ktot = (seq_len + kRows - 1) / kRows;
  const int npair = (ktot + 1) / 2, items = npair * batch * heads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tkv);
    for (int i = 0; i < 11; ++i) mbar_init(bars + i, 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&p_full[t], 128);
      mbar_init(&pv_done[t], 1);
      mbar_init(&s_free[t], 128);
      mbar_init(&o_free[t], 128);
    }
    mbar_init(q_empty, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA: Q_A, Q_B, then the K ring ----------------
      uint32_t kc = 0;  // K loads issued by this CTA
      for (int n = 0; n * static_cast<int>(gridDim.x) < items; ++n) {  // n = items done (all rounds but the last are full)
        const int w = item_of(n, blockIdx.x, gridDim.x);
        if (w >= items) continue;
        const Item it = item_at(w, npair, heads, ktot);
        if (n >= 1) wait_bar(q_empty, (n - 1) & 1, 11, n);
        mbar_arrive_expect_tx(q_full, 2 * C::kTile);
        for (int t = 0; t < 2; ++t)
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(base + C::kQ + t * C::kTile + c * C::kBox, &tq, q_full, it.hd * D + c * 64, it.b,
                        (2 * it.pair + t) * kRows);
        for (int j = 0; j < it.ntk; ++j, ++kc) {
          const uint32_t st = kc % kKS;
          if (kc >= kKS) wait_bar(&k_empty[st], ((kc - kKS) / kKS) & 1, 1, j);
          mbar_arrive_expect_tx(&k_full[st], C::kTile);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(base + C::kK + st * C::kTile + c * C::kBox, &tkv, &k_full[st], it.hd * D + c * 64, it.b,
                        j * kRows);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {  // ---------------- TMA: the V ring ----------------
      uint32_t vc = 0;
      for (int n = 0; n * static_cast<int>(gridDim.x) < items; ++n) {
        const int w = item_of(n, blockIdx.x, gridDim.x);
        if (w >= items) continue;
        const Item it = item_at(w, npair, heads, ktot);
        for (int j = 0; j < it.ntk; ++j, ++vc) {
          const uint32_t st = vc % VS;
          if (vc >= VS) wait_bar(&v_empty[st], ((vc - VS) / VS) & 1, 2, j);
          mbar_arrive_expect_tx(&v_full[st], C::kTile);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(base + C::kV + st * C::kTile + c * C::kBox, &tkv, &v_full[st], it.hd * D + c * 64,
                        batch + it.b, j * kRows);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_s = umma_idesc_f16_f32(kRows, kRows);
      constexpr uint32_t idesc_o = umma_idesc_f16_f32(kRows, D) | (1u << 16);  // B (V) MN-major
      uint32_t kc = 0, vc = 0;            // K / V tiles consumed
      uint32_t sc[2] = {0, 0}, pc[2] = {0, 0};  // S_t issued, P_t consumed (running over items)
      for (int n = 0; n * static_cast<int>(gridDim.x) < items; ++n) {
        const int w = item_of(n, blockIdx.x, gridDim.x);
        if (w >= items) continue;
        const Item it = item_at(w, npair, heads, ktot);
        wait_bar(q_full, n & 1, 3, n);
        for (int j = 0; j <= it.ntk; ++j) {
          if (j < it.ntk) {
            const uint32_t st = kc % kKS;
            wait_bar(&k_full[st], (kc / kKS) & 1, 6, j);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              if (j < (t ? it.ntk : it.nt_a)) {  // S_t(j) once softmax t holds its previous S in registers
                if (sc[t] >= 1) wait_bar(&s_free[t], (sc[t] - 1) & 1, 4, j);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < D / 64; ++c)
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    umma_f16(tmem + t * kRows, umma_desc_k_sw128(base + C::kQ + t * C::kTile + c * C::kBox + k * 32),
                             umma_desc_k_sw128(base + C::kK + st * C::kTile + c * C::kBox + k * 32), idesc_s,
                             (c | k) != 0);
                umma_commit(&s_full[t]);
                ++sc[t];
              }
            }
            umma_commit(&k_empty[st]);  // both tiles' S on K_j issued before
            ++kc;
            if (j == it.ntk - 1) umma_commit(q_empty);  // the item's last S MMAs: Q may be reloaded
          }
          if (j >= 1) {
            const uint32_t st = vc % VS;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              if (j - 1 < (t ? it.ntk : it.nt_a)) {  // O_t += P_t(j-1) V_{j-1} once P_t(j-1) is in smem
                wait_bar(&p_full[t], pc[t] & 1, 10, j);
                if (j == 1 && n >= 1) wait_bar(&o_free[t], (n - 1) & 1, 12, n);  // previous item's O_t read
                wait_bar(&v_full[st], (vc / VS) & 1, 5, j);
                tc_fence_after();
                const uint32_t p = base + C::kP + t * C::kP1;
#pragma unroll
                for (int kk = 0; kk < kRows / 16; ++kk)
                  umma_f16(tmem + C::kO + t * D, umma_desc_k_sw128(p + (kk >> 2) * C::kBox + (kk & 3) * 32),
                           desc_mn_sw128(base + C::kV + st * C::kTile + kk * 2048, C::kBox), idesc_o,
                           (j - 1 | kk) != 0);
                umma_commit(&pv_done[t]);
                ++pc[t];
              }
            }
            umma_commit(&v_empty[st]);  // both tiles' P V on V_{j-1} issued before
            ++vc;
          }
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- softmax, O correction, epilogue of tile t ----------------
    const int t = (warp - 4) >> 2;
    const int tt = threadIdx.x - 128 * (t + 1);
    const uint32_t lanes = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    const uint32_t s_col = tmem + lanes + t * kRows, o_col = tmem + lanes + C::kO + t * D;
    const uint32_t p_base = base + C::kP + t * C::kP1;
    uint32_t sc = 0, pc = 0;  // S_t(.) received, P V of tile t done (running over items)
    for (int n = 0; n * static_cast<int>(gridDim.x) < items; ++n) {
      const int w = item_of(n, blockIdx.x, gridDim.x);
      if (w >= items) continue;
      const Item it = item_at(w, npair, heads, ktot);
      const int qt = 2 * it.pair + t, row = qt * kRows + tt, ntt = t ? it.ntk : it.nt_a;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < ntt; ++j) {
        wait_bar(&s_full[t], sc & 1, 7, j);
        ++sc;
        tc_fence_after();
        uint32_t r[kRows];  // this row's raw scores Q K^T (the scale is folded into exp2 below)
#pragma unroll
        for (int cc = 0; cc < kRows / 32; ++cc)
          tmem_ld_32x32b_x32(s_col + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&s_free[t]);  // the MMA may now compute S_t(j+1) under this tile's softmax
        if (j == qt) {  // diagonal tile (warp-uniform branch): keys past the query (and past seq_len) masked
          const int lim = row - j * kRows;
#pragma unroll
          for (int i = 0; i < kRows; ++i)
            if (i > lim) r[i] = __float_as_uint(-INFINITY);
        }
        float mx = row_max128(r) * qscale;  // qscale > 0: the max of the scaled scores (finite: key j*128 <= row)
        // lazy rescaling: keep the running max unless this tile exceeds it by more than 2^8 (P <= 256
        // stays exact enough in fp16 and O / l absorb the common factor), so most tiles after the first
        // skip the O correction; the first tile always sets it
        mx = (mx > m + 8.f) ? mx : m;
        const float alpha = ex2_approx(m - mx);
        if (j >= 1) {  // P V of the previous tile is done: O_t and the P_t buffer are ours
          wait_bar(&pv_done[t], pc & 1, 8, j);
          ++pc;
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {  // warp-uniform: tcgen05.ld/st are .sync.aligned
#pragma unroll 1
            for (int cc = 0; cc < D / 16; ++cc) {
              uint32_t o[16];
              tmem_ld_x16(o_col + cc * 16, o);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st_x16(o_col + cc * 16, o);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          }
        }
        l = l * alpha + exp_store128(r, qscale, mx, p_base, tt, C::kBox);
        m = mx;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy P writes -> tcgen05 reads
        tc_fence_before();
        mbar_arrive(&p_full[t]);
      }
      wait_bar(&pv_done[t], pc & 1, 9, ntt);  // the item's last P V (also frees P_t for the next item)
      ++pc;
      tc_fence_after();
      const float inv = 1.f / l;
      __half* o = out + (static_cast<long long>(row) * batch + it.b) * heads * D + it.hd * D;
#pragma unroll 1
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(o_col + cc * 32, r);
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
      tc_fence_before();
      mbar_arrive(&o_free[t]);  // O_t read out: the next item's first P V may overwrite it
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
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
  static int sms[64] = {0};
  if (dev < 64 && sms[dev] == 0) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const long long items = static_cast<long long>((seq_len + 2 * tc::kRows - 1) / (2 * tc::kRows)) * batch * heads;
  const int nsm = dev < 64 && sms[dev] > 0 ? sms[dev] : 148;
  const int grid = static_cast<int>(items < nsm ? items : nsm);  // persistent: one CTA per SM
  tc::prefill_tc_kernel<D><<<grid, 384, C::kSmem, stream>>>(tq, tkv, out, batch, heads, seq_len, qscale);
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
