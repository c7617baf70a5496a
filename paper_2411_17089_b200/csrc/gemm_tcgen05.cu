// K1 and every other dense projection on the decode path: a persistent,
// warp-specialised tcgen05 GEMM for sm_100a.
//
//   D[m, n] = epilogue( sum_k A[m, k] * W[n, k] + bias[n] )
//
// A (activations, fp16, K-major) and W (weights, fp16, K-major, i.e. the
// PyTorch Linear layout [out, in]) are streamed by TMA into a STAGES-deep
// ring of 128B-swizzled shared-memory tiles.  One elected thread issues
// tcgen05.mma (M=128, N=BN, K=16) into a double-buffered TMEM accumulator;
// four epilogue warps drain TMEM with tcgen05.ld, add the bias, apply the
// optional scale/ReLU/residual, convert, and scatter rows straight into the
// caller's layout — for K1 that is the position-major KV page buffer, so the
// recompute writes K and V where attention will read them with no separate
// copy or cast kernel (reference semantics: numerics.py:129-137,
// costmodel.py:169-176).
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w3 idle, w4..w7 epilogue (warp w%4 owns TMEM lanes [32*(w%4), +32)).

#include <stdlib.h>

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of fp16 along K
constexpr int kBnSwapAB = -1;  // gemm_f16 tile code of the swapped-operand decode GEMM
constexpr int kBnGemv = -2;    // CUDA-core decode projection, M <= kGemvMaxM (gemv.cu)
constexpr long long kABandBytes = 32ll << 20;
constexpr int kSkMaxTiles = 4096;

// KVPR_GEMM_TRACE (tools only): per-CTA globaltimer stamps of the swap-AB decode GEMM
__device__ unsigned long long* g_gemm_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// compiled in only with -DKVPR_GEMM_TRACE: even a null check of the pointer is an L2 load on the
// epilogue's critical path
__device__ __forceinline__ void gstamp(int slot) {
#ifdef KVPR_GEMM_TRACE
  if (g_gemm_trace != nullptr) g_gemm_trace[blockIdx.x * 8 + slot] = gtimer();
#else
  (void)slot;
#endif
}  // stream-K: n tiles of 128 outputs per decode GEMM (N <= 524288)

// The 1-CTA ring is sized at launch: stage = A box (a_box_rows x 128 B: 16 KB, or only the live
// rows of a small-M decode GEMM) + B box (BN x 128 B), as many stages as fit in shared memory
// (<= kMaxStages).  A decode GEMM (M = batch) is weight streaming: its per-CTA rate is the
// weight bytes in flight / the TMA round trip, so the ring holds only live A rows and spends the
// rest of the 227 KB on B.  The MMA still reads a 128-row A operand; rows past a_box_rows fall on
// the next stages' bytes (inside the allocation), which only feed accumulator rows >= M that the
// epilogue never stores.
constexpr int kMaxStages = 48;
constexpr uint32_t kSmemBudget = 227 * 1024;
constexpr uint32_t kBarrierBytes = 1024;

template <int BN>
struct GemmCfg {
  static constexpr uint32_t kABytes = kBM * kBK * 2;  // full 128-row A box
  static constexpr uint32_t kBBytes = BN * kBK * 2;
  static constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr uint32_t kSmemBytes = kSmemBudget;
};

// stages that fit: 1024 B alignment slack + barriers + stages x (A + B), and the last A stage's
// 128-row MMA read (16 KB) stays inside the allocation
__host__ __device__ inline int ring_stages(uint32_t a_stage, uint32_t b_stage) {
  int s = static_cast<int>((kSmemBudget - 1024 - kBarrierBytes) / (a_stage + b_stage));
  return s < kMaxStages ? s : kMaxStages;
}


// Epilogue for one thread: 32 fp32 accumulators of row (r_in, r_grp) at columns [n0, n0+32):
// + bias, optional scale / ReLU, convert, scatter into the caller's layout (see GemmArgs).
__device__ __forceinline__ void store_chunk_f(const GemmArgs& p, float (&v)[32], int n0, long long r_in,
                                              long long r_grp) {
  if (p.bias != nullptr) {
    const uint4* bp = reinterpret_cast<const uint4*>(p.bias + n0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint4 bw = __ldg(bp + u);
      const __half2* h2 = reinterpret_cast<const __half2*>(&bw);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __half22float2(h2[e]);
        v[u * 8 + e * 2] += f.x;
        v[u * 8 + e * 2 + 1] += f.y;
      }
    }
  }
  if (n0 < p.scale_cols) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= p.scale;
  }
  if (p.flags & KVPR_EPI_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  const int seg = n0 / p.seg_width;
  const int col = n0 - seg * p.seg_width;
  // select the segment without dynamic indexing of the param arrays (keeps them out of local memory)
  void* sp = seg == 0 ? p.seg_ptr[0] : (seg == 1 ? p.seg_ptr[1] : p.seg_ptr[2]);
  const long long gs = seg == 0 ? p.seg_group_stride[0] : (seg == 1 ? p.seg_group_stride[1] : p.seg_group_stride[2]);
  const long long off = r_in * p.ld + r_grp * gs + col;
  if (p.flags & KVPR_EPI_F32) {
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(sp) + off);
    if (p.flags & KVPR_EPI_ACCUM) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4 old = o[u];
        old.x += v[u * 4 + 0];
        old.y += v[u * 4 + 1];
        old.z += v[u * 4 + 2];
        old.w += v[u * 4 + 3];
        o[u] = old;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) o[u] = make_float4(v[u * 4], v[u * 4 + 1], v[u * 4 + 2], v[u * 4 + 3]);
    }
  } else {
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(sp) + off);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint4 w;
      w.x = pack_half2(v[u * 8 + 0], v[u * 8 + 1]);
      w.y = pack_half2(v[u * 8 + 2], v[u * 8 + 3]);
      w.z = pack_half2(v[u * 8 + 4], v[u * 8 + 5]);
      w.w = pack_half2(v[u * 8 + 6], v[u * 8 + 7]);
      o[u] = w;
    }
  }
}

__device__ __forceinline__ void store_chunk(const GemmArgs& p, const uint32_t (&r)[32], int n0, int row,
                                            long long r_in, long long r_grp, int ks) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (p.k_splits > 1) {  // raw partial of this K slice; split_k_reduce applies the epilogue
    float4* o = reinterpret_cast<float4*>(p.ws + (static_cast<long long>(ks) * p.M + row) * p.ws_ld + n0);
#pragma unroll
    for (int u = 0; u < 8; ++u) o[u] = make_float4(v[u * 4], v[u * 4 + 1], v[u * 4 + 2], v[u * 4 + 3]);
    return;
  }
  store_chunk_f(p, v, n0, r_in, r_grp);
}

// Deterministic split-K reduction: partials summed in slice order, then the GEMM epilogue.
__global__ void split_k_reduce_kernel(const GemmArgs p) {
  pdl_trigger();
  pdl_wait();
  const int chunks = p.N / 32;
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(p.M) * chunks) return;
  const int row = static_cast<int>(t / chunks);
  const int n0 = static_cast<int>(t % chunks) * 32;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = 0.f;
  for (int ks = 0; ks < p.k_splits; ++ks) {
    const float4* w = reinterpret_cast<const float4*>(p.ws + (static_cast<long long>(ks) * p.M + row) * p.ws_ld + n0);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 x = w[u];
      v[u * 4] += x.x;
      v[u * 4 + 1] += x.y;
      v[u * 4 + 2] += x.z;
      v[u * 4 + 3] += x.w;
    }
  }
  store_chunk_f(p, v, n0, row % p.row_group, row / p.row_group);
}

// Tile order.  group > 0: bands of `group` m-blocks, n-major inside a band, so the CTAs in flight
// share the band's A (reused across n from L2) while B streams past once per band.  group < 0:
// bands of -group n-blocks, m-major inside, so the band's B stays in L2 while A streams once per
// band.  The host picks the orientation with fewer DRAM reads and sizes the band to stay
// L2-resident (kABandBytes: 16 pair blocks = 32 MB at K = 4096 measured best; 24 or all thrash).
// Odd bands sweep backwards, so a band starts on the blocks the previous one just left in L2.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int group, int& m_blk, int& n_blk) {
  if (group > 0) {
    const int per_group = group * num_n;
    const int g = tile / per_group;
    const int first_m = g * group;
    const int gm = min(group, num_m - first_m);
    const int local = tile - g * per_group;
    m_blk = first_m + local % gm;
    n_blk = (g & 1) ? num_n - 1 - local / gm : local / gm;
  } else {
    const int gsz = -group;
    const int per_group = gsz * num_m;
    const int g = tile / per_group;
    const int first_n = g * gsz;
    const int gn = min(gsz, num_n - first_n);
    const int local = tile - g * per_group;
    n_blk = first_n + local % gn;
    m_blk = (g & 1) ? num_m - 1 - local / gn : local / gn;
  }
}

template <int BN>
__global__ void __launch_bounds__(256, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const GemmArgs p) {
  using Cfg = GemmCfg<BN>;
  const uint32_t a_stage = static_cast<uint32_t>(p.a_box_rows) * kBK * 2;
  const int STAGES = ring_stages(a_stage, Cfg::kBBytes);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * a_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::kBBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int splits = p.k_splits > 1 ? p.k_splits : 1;
  const int num_tiles = p.num_m_blk * p.num_n_blk * splits;
  const int kb_per = (p.num_k_blk + splits - 1) / splits;  // host guarantees every slice is non-empty

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      // The weights (B) never depend on an earlier kernel: the first ring's worth of B boxes is
      // issued before the PDL wait, so the weight stream starts under the previous kernel's tail;
      // A (activations) and everything after follow the wait.
      // small-M GEMMs load only the live rows of A; the rest of the 128-row operand is stale smem
      // that only produces accumulator rows the epilogue never stores
      uint32_t stage = 0, phase = 0;
      int it = 0, pre = 0;
      for (int pass = 0; pass < 3; ++pass) {  // 0: B prefetch, 1: A of the prefetched, 2: the rest
        if (pass == 1) pdl_wait();
        it = 0;
        stage = 0;
        phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
          int m_blk, n_blk;
          tile_coords(tile / splits, p.num_m_blk, p.num_n_blk, p.group_m, m_blk, n_blk);
          const int kb0 = (tile % splits) * kb_per;
          const int kb1 = min(p.num_k_blk, kb0 + kb_per);
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            if (pass == 0 && it == STAGES) break;
            if (pass == 1 && it == pre) break;
            if (pass == 2 && it < pre) {
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
              continue;
            }
            if (pass != 1) {
              mbar_wait(&empty[stage], phase ^ 1);
              mbar_arrive_expect_tx(&full[stage], a_stage + Cfg::kBBytes);
              tma_load_2d(sB + stage * Cfg::kBBytes, &tmap_b, &full[stage], kb * kBK, n_blk * BN);
            }
            if (pass != 0) tma_load_2d(sA + stage * a_stage, &tmap_a, &full[stage], kb * kBK, m_blk * kBM);
            if (pass == 0) ++pre;
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if ((pass == 0 && it == STAGES) || (pass == 1 && it == pre)) break;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread) ----------------
      constexpr uint32_t idesc = umma_idesc_f16_f32(kBM, BN);
      uint32_t stage = 0, phase = 0, local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const uint32_t acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb0 = (tile % splits) * kb_per;
        const int kb1 = min(p.num_k_blk, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * a_stage);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // advancing K by 16 fp16 = 32 bytes inside the 128B swizzle atom
            umma_f16(d_tmem, umma_desc_k_sw128(a_addr + k * 32), umma_desc_k_sw128(b_addr + k * 32), idesc,
                     (kb != kb0) || (k != 0));
          }
          umma_commit(&empty[stage]);  // frees this smem slot once the MMAs above retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> regs -> global ----------------
    pdl_wait();  // the residual (ACCUM) and every output buffer belong to the preceding kernels
    const uint32_t q = warp & 3;
    uint32_t local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      int m_blk, n_blk;
      tile_coords(tile / splits, p.num_m_blk, p.num_n_blk, p.group_m, m_blk, n_blk);
      const int ks = tile % splits;
      const uint32_t acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * kBM + q * 32 + lane;
      const bool row_ok = row < p.M;
      // row -> (group, offset) once per tile
      const long long r_in = row_ok ? (row % p.row_group) : 0;
      const long long r_grp = row_ok ? (row / p.row_group) : 0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        __syncwarp();
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((q * 32u) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int n0 = n_blk * BN + c * 32;
        if (!row_ok || n0 >= p.N) continue;
        store_chunk(p, r, n0, row, r_in, r_grp, ks);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}


// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for the large-M GEMMs (K1, prefill): a
// cluster of 2 CTAs computes a 256 x 256 tile with one tcgen05.mma M=256
// issued by the leader.  Each CTA stages its 128-row half of A and its
// 128-row half of B (so per-SM smem/L2 operand traffic drops by a third vs the
// 1-CTA 128x256 tile) in a 6-deep ring; each CTA's TMEM holds the 128 x 256
// accumulator of its own rows (double buffered, 512 columns).
//   full[s]   (leader)  : leader arrive.expect_tx(both CTAs' bytes) + both CTAs' TMA complete_tx
//   empty[s]  (both)    : leader's tcgen05.commit multicast to the pair
//   tfull[a]  (both)    : leader's commit multicast after the last k-block of a tile
//   tempty[a] (leader)  : 8 epilogue warps (4 per CTA) arrive, the peer's remotely

constexpr int k2BN = 256;             // N of the pair tile (each CTA stages 128 rows of B)
constexpr int k2Stages = 6;
constexpr uint32_t k2ABytes = kBM * kBK * 2;          // 16 KB: this CTA's 128 rows of A
constexpr uint32_t k2BBytes = (k2BN / 2) * kBK * 2;   // 16 KB: this CTA's 128 rows of B
constexpr uint32_t k2StageBytes = k2ABytes + k2BBytes;
constexpr uint32_t k2SmemBytes = k2Stages * k2StageBytes + 1024 + 256;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_tcgen05_2sm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                            const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + k2Stages * k2ABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + k2Stages * k2BBytes);
  uint64_t* empty = full + k2Stages;
  uint64_t* tfull = empty + k2Stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = p.num_m_blk * p.num_n_blk;
  const int num_kb = p.num_k_blk;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      // same PDL split as the 1-CTA producer: first ring of W_kv boxes before the wait
      uint32_t stage = 0, phase = 0;
      int it = 0, pre = 0;
      for (int pass = 0; pass < 3; ++pass) {  // 0: B prefetch, 1: A of the prefetched, 2: the rest
        if (pass == 1) pdl_wait();
        it = 0;
        stage = 0;
        phase = 0;
        for (int tile = cluster; tile < num_tiles; tile += nclusters) {
          int m_blk, n_blk;
          tile_coords(tile, p.num_m_blk, p.num_n_blk, p.group_m, m_blk, n_blk);
          const int a_row = m_blk * 2 * kBM + rank * kBM;
          const int b_row = n_blk * k2BN + rank * (k2BN / 2);
          for (int kb = 0; kb < num_kb; ++kb, ++it) {
            if (pass == 0 && it == k2Stages) break;
            if (pass == 1 && it == pre) break;
            if (pass == 2 && it < pre) {
              if (++stage == k2Stages) {
                stage = 0;
                phase ^= 1;
              }
              continue;
            }
            if (pass != 1) {
              mbar_wait(&empty[stage], phase ^ 1);
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * k2StageBytes);
              tma_load_2d_2sm(sB + stage * k2BBytes, &tmap_b, &full[stage], kb * kBK, b_row);
            }
            if (pass != 0) tma_load_2d_2sm(sA + stage * k2ABytes, &tmap_a, &full[stage], kb * kBK, a_row);
            if (pass == 0) ++pre;
            if (++stage == k2Stages) {
              stage = 0;
              phase ^= 1;
            }
          }
          if ((pass == 0 && it == k2Stages) || (pass == 1 && it == pre)) break;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader CTA, single thread) ----------------
      constexpr uint32_t idesc = umma_idesc_f16_f32(2 * kBM, k2BN);
      uint32_t stage = 0, phase = 0, local = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters, ++local) {
        const uint32_t acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * k2BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * k2ABytes);
          const uint32_t b_addr = smem_u32(sB + stage * k2BBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            umma_f16_2sm(d_tmem, umma_desc_k_sw128(a_addr + k * 32), umma_desc_k_sw128(b_addr + k * 32), idesc,
                         (kb | k) != 0);
          }
          umma_commit_2sm(&empty[stage], 0x3);
          if (++stage == k2Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2sm(&tfull[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, own 128 rows) ----------------
    pdl_wait();
    const uint32_t q = warp & 3;
    uint32_t local = 0;
    for (int tile = cluster; tile < num_tiles; tile += nclusters, ++local) {
      int m_blk, n_blk;
      tile_coords(tile, p.num_m_blk, p.num_n_blk, p.group_m, m_blk, n_blk);
      const uint32_t acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * 2 * kBM + rank * kBM + q * 32 + lane;
      const bool row_ok = row < p.M;
      const long long r_in = row_ok ? (row % p.row_group) : 0;
      const long long r_grp = row_ok ? (row / p.row_group) : 0;
#pragma unroll 1
      for (int c = 0; c < k2BN / 32; ++c) {
        __syncwarp();
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((q * 32u) << 16) + acc * k2BN + c * 32, r);
        tmem_ld_wait();
        const int n0 = n_blk * k2BN + c * 32;
        if (!row_ok || n0 >= p.N) continue;
        store_chunk(p, r, n0, row, r_in, r_grp, 0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty[acc]);
        else
          mbar_arrive_remote(&tempty[acc], 0);
      }
    }
  }

  tc_fence_before();
  cluster_sync();  // no MMA in flight, both epilogues done
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// Weight-streaming decode GEMM (M = batch rows <= 64): operands swapped.
//
//   D^T[n, m] = sum_k W[n, k] * A[m, k]
//
// A decode GEMM has a handful of live activation rows against megabytes of weights.  In the
// regular kernel the activations are the MMA's M operand, padded to 128 rows, and the weights
// the N operand: a k-block then costs a full 128 x BN MMA for 4..32 useful rows, and one CTA's
// chain of dependent MMAs, not HBM, sets the pace (~0.25 us per 64-wide k-block whatever BN).
// Here the weight tile is the 128-row M operand and the activation rows the N operand (MP = M
// rounded up to 16; TMA zero-fills rows >= M), so every k-block of the same MMA chain moves 16 KB
// of weights and the tensor core does no padded work on the weight side.  The accumulator is
// 128 TMEM lanes (weight rows) x MP columns (activation rows); the epilogue thread owning lane
// n writes column n of every output row m (coalesced across the warp for each m).
//
// The k order per output element is the regular kernel's (k-blocks ascending, 16-wide MMA K
// steps), so an unsplit launch reproduces it bit for bit (tested against K1: the decode-time
// k, v of the new token must equal the K1 rebuild).  With a workspace (never for the q/k/v
// projection) the kernel runs stream-K: every SM streams an equal share of the k-block units, and
// tiles shared by several CTAs are finished in-kernel by the last CTA to arrive, which sums the
// fp32 partial slots in k order (deterministic) and applies the epilogue -- no reduce launch.

constexpr uint32_t kSwWBytes = kBM * kBK * 2;  // 16 KB: 128 weight rows x 64 k

// KB 64-wide k-boxes per ring stage: a stage reads KB x 128 B contiguous from each of its 128
// weight rows (one DRAM page visit instead of KB), at the cost of fewer, larger stages.
template <int MP, int KB>
struct SwapCfg {
  static constexpr uint32_t kXBox = MP * kBK * 2;
  static constexpr uint32_t kWStage = KB * kSwWBytes;
  static constexpr uint32_t kXStage = KB * kXBox;
  static constexpr uint32_t kStageBytes = kWStage + kXStage;
  static constexpr int kStages = static_cast<int>((kSmemBudget - 1024 - kBarrierBytes) / kStageBytes) < kMaxStages
                                     ? static_cast<int>((kSmemBudget - 1024 - kBarrierBytes) / kStageBytes)
                                     : kMaxStages;
  static constexpr uint32_t kTmemCols = (2 * MP <= 32) ? 32 : (2 * MP <= 64 ? 64 : 128);
};

template <int MP>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[MP]);

template <>
__device__ __forceinline__ void tmem_ld_cols<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <>
__device__ __forceinline__ void tmem_ld_cols<32>(uint32_t taddr, uint32_t (&r)[32]) {
  tmem_ld_32x32b_x32(taddr, r);
}

template <>
__device__ __forceinline__ void tmem_ld_cols<64>(uint32_t taddr, uint32_t (&r)[64]) {
  tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
  tmem_ld_32x32b_x32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
}

// Work of one CTA as a list of segments (n block, k-blocks [kb0, kb1)).
//  * stream-K (p.sk_ctas > 0): the n_blk x num_k_blk k-block units are cut into sk_ctas equal
//    contiguous ranges, one per CTA, so every SM streams the same number of weight bytes whatever
//    the tile count (out-proj: 32 tiles -> 148 CTAs of 13-14 k-blocks).  A range covers the tail of
//    one tile, whole tiles, and the head of another.
//  * otherwise: whole tiles, grid-strided (the q/k/v projection, whose k, v must carry K1's bits, and
//    the TP push).
struct SegIter {
  int u, u_end, tile, stride, n_blk_count, nkb;
  bool sk;
  __device__ SegIter(const GemmArgs& p) {
    nkb = p.num_k_blk;
    n_blk_count = p.num_n_blk;
    sk = p.sk_ctas > 0;
    if (sk) {
      const long long U = static_cast<long long>(p.num_n_blk) * nkb;
      u = static_cast<int>(U * blockIdx.x / p.sk_ctas);
      u_end = static_cast<int>(U * (blockIdx.x + 1) / p.sk_ctas);
    } else {
      tile = blockIdx.x;
      stride = gridDim.x;
    }
  }
  // next segment; first = it is the CTA's first one (the partial slot convention below)
  __device__ bool next(int& n_blk, int& kb0, int& kb1) {
    if (sk) {
      if (u >= u_end) return false;
      n_blk = u / nkb;
      kb0 = u - n_blk * nkb;
      kb1 = min(nkb, kb0 + (u_end - u));
      u += kb1 - kb0;
      return true;
    }
    if (tile >= n_blk_count) return false;
    n_blk = tile;
    kb0 = 0;
    kb1 = nkb;
    tile += stride;
    return true;
  }
};

// Barrier of the 128 epilogue threads (named barrier 1) that also ORs a predicate over them: how
// thread 128's arrival verdict reaches the others without a shared flag (a flag rewritten for the next
// segment could race a slow reader of the previous one; compute-sanitizer racecheck flagged it)
__device__ __forceinline__ bool epi_bar_or(bool v) {
  unsigned r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %1, 0;\n\tbar.red.or.pred p, 1, 128, q;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(static_cast<unsigned>(v))
      : "memory");
  return r != 0;
}

// stream-K bookkeeping for tile t: the CTAs whose unit ranges meet it are [c_first, c_last]
// (range of CTA c = [floor(c U / G), floor((c+1) U / G))); CTA c's segment of t sits in partial slot
// 2c if c's range starts inside t (its first segment), else 2c + 1 (its last).
__device__ __forceinline__ int sk_cta_of_unit(long long x, long long U, int G) {
  // largest c with floor(c U / G) <= x
  const long long c = ((x + 1) * G - 1) / U;
  return static_cast<int>(c < G - 1 ? c : G - 1);
}

template <int MP, int KB>
__global__ void __launch_bounds__(256, 1)
    gemm_swapab_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
                       const GemmArgs p) {
  using Cfg = SwapCfg<MP, KB>;
  constexpr int STAGES = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * Cfg::kWStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + STAGES * Cfg::kXStage);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  pdl_trigger();
  if (threadIdx.x == 0) gstamp(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: weights before the PDL wait, activations after ----------------
      // pass 0 issues the first ring of WEIGHT boxes (they never depend on an earlier kernel), pass 1
      // (after the wait) their activation boxes, pass 2 everything after
      uint32_t stage = 0, phase = 0;
      int it = 0, pre = 0;
      for (int pass = 0; pass < 3; ++pass) {
        if (pass == 1) pdl_wait();
        it = 0;
        stage = 0;
        phase = 0;
        SegIter segs(p);
        int n_blk, kb0, kb1;
        bool stop = false;
        while (!stop && segs.next(n_blk, kb0, kb1)) {
          for (int kb = kb0; kb < kb1; kb += KB, ++it) {
            if ((pass == 0 && it == STAGES) || (pass == 1 && it == pre)) {
              stop = true;
              break;
            }
            if (pass == 2 && it < pre) {
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
              continue;
            }
            const int nbox = min(KB, kb1 - kb);
            if (pass != 1) {
              mbar_wait(&empty[stage], phase ^ 1);
              mbar_arrive_expect_tx(&full[stage], nbox * (kSwWBytes + Cfg::kXBox));
              for (int j = 0; j < nbox; ++j) {
                // tiled weights: box (n_blk, kb) is the 16 KB contiguous run of rows (n_blk * nkb + kb) * 128
                // of a [*, 64] matrix, so a CTA streams one contiguous region (DRAM-page friendly)
                if (p.w_tiled)
                  tma_load_2d(sW + stage * Cfg::kWStage + j * kSwWBytes, &tmap_w, &full[stage], 0,
                              (n_blk * p.num_k_blk + kb + j) * kBM);
                else
                  tma_load_2d(sW + stage * Cfg::kWStage + j * kSwWBytes, &tmap_w, &full[stage], (kb + j) * kBK,
                              n_blk * kBM);
              }
            }
            if (pass != 0) {
              for (int j = 0; j < nbox; ++j)
                tma_load_2d(sX + stage * Cfg::kXStage + j * Cfg::kXBox, &tmap_x, &full[stage], (kb + j) * kBK, 0);
            }
            if (pass == 0) ++pre;
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: M = 128 weight rows, N = MP activation rows ----------------
      constexpr uint32_t idesc = umma_idesc_f16_f32(kBM, MP);
      uint32_t stage = 0, phase = 0, local = 0;
      SegIter segs(p);
      int n_blk, kb0, kb1;
      while (segs.next(n_blk, kb0, kb1)) {
        const uint32_t acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        ++local;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * MP;
        for (int kb = kb0; kb < kb1; kb += KB) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const int nbox = min(KB, kb1 - kb);
          for (int j = 0; j < nbox; ++j) {
            const uint32_t w_addr = smem_u32(sW + stage * Cfg::kWStage + j * kSwWBytes);
            const uint32_t x_addr = smem_u32(sX + stage * Cfg::kXStage + j * Cfg::kXBox);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              umma_f16(d_tmem, umma_desc_k_sw128(w_addr + k * 32), umma_desc_k_sw128(x_addr + k * 32), idesc,
                       (kb != kb0) || (j != 0) || (k != 0));
            }
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: lane n of the tile, every activation row m ----------------
    pdl_wait();
    const uint32_t q = warp & 3;
    uint32_t local = 0;
    SegIter segs(p);
    int n_blk, kb0, kb1;
    while (segs.next(n_blk, kb0, kb1)) {
      const bool first_seg = local == 0;
      const uint32_t acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ++local;
      mbar_wait(&tfull[acc], acc_phase);
      if (threadIdx.x == 128 && local <= 3) gstamp(local);
      tc_fence_after();
      uint32_t r[MP];
      tmem_ld_cols<MP>(tmem_base + ((q * 32u) << 16) + acc * MP, r);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);  // accumulator drained into registers
      const int col = q * 32 + lane;               // column inside the 128-wide tile
      const int n = n_blk * kBM + col;
      if (p.tp_world > 1) {
        // fused TP all-reduce, push half (csrc/tpcomm.cu): the raw fp32 partial of this tile goes
        // straight into slot [rank] of the tile owner's receive buffer over NVLink, then the owner's
        // flag for (rank, tile) is released at system scope
        const int owner = n_blk % p.tp_world;
        if (n < p.N) {
          float* o = p.tp_recv[owner] + static_cast<long long>(p.tp_rank) * p.M * p.N + n;
#pragma unroll
          for (int m = 0; m < MP; ++m)
            if (m < p.M) o[static_cast<long long>(m) * p.N] = __uint_as_float(r[m]);
        }
        __threadfence_system();
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps of this tile
        if (threadIdx.x == 128) {
          unsigned* f = p.tp_flags[owner] + p.tp_rank * kTpMaxTiles + n_blk;
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(p.tp_epoch) : "memory");
        }
        continue;
      }
      float v[MP];
#pragma unroll
      for (int m = 0; m < MP; ++m) v[m] = __uint_as_float(r[m]);
      if (kb0 != 0 || kb1 != p.num_k_blk) {
        // stream-K partial tile.  Every contributor but the last stores its raw fp32 partial in a slot
        // and counts itself in; the last one to arrive sums all partials in k order (deterministic:
        // the order never depends on which CTA finishes last) and applies the epilogue.  The CTA
        // holding a tile's first k-blocks (c_first) usually reaches it last -- the tile is its final
        // segment, while for every later CTA it is the first -- so it checks the count before
        // publishing: if the others are all in, it keeps its partial in registers and skips a slot
        // store and an atomic round trip on the kernel's critical tail.
        const long long U = static_cast<long long>(p.num_n_blk) * p.num_k_blk;
        const int G = p.sk_ctas;
        const int c = blockIdx.x;
        const long long t0 = static_cast<long long>(n_blk) * p.num_k_blk;
        const int c_first = sk_cta_of_unit(t0, U, G);
        const int c_last = sk_cta_of_unit(t0 + p.num_k_blk - 1, U, G);
        const unsigned others = static_cast<unsigned>(c_last - c_first);
        unsigned* ctr = p.sk_counters + n_blk;
        bool last = false;
        if (c == c_first && !first_seg) {
          bool seen_all = false;
          if (threadIdx.x == 128) {
            unsigned seen;
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
            seen_all = seen == others;
            if (seen_all) *ctr = 0u;  // every other arrival of this launch is in: zero for the next call
          }
          last = epi_bar_or(seen_all);  // thread 128's verdict to all 128 epilogue threads
        }
        if (!last) {
          float* slot = p.ws + (2LL * c + (first_seg ? 0 : 1)) * MP * kBM;
#pragma unroll
          for (int m = 0; m < MP; ++m) slot[m * kBM + col] = v[m];
          // publish: the CTA barrier orders the 128 threads' slot stores before thread 128's arrival,
          // a gpu-scope acq_rel atomic (release is cumulative); the last arriver's acquire + the
          // second barrier order every slot before the reads below
          asm volatile("bar.sync 1, 128;" ::: "memory");
          bool fin = false;
          if (threadIdx.x == 128) {
            unsigned old;
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
            fin = old == others;
            if (fin) *ctr = 0u;
          }
          if (!epi_bar_or(fin)) continue;
        }
        const bool own_in_regs = last;  // c_first's partial never went to its slot
        if (threadIdx.x == 128) gstamp(4);
        // sum the slots in k order (CTA c_first's is its last segment, every later CTA's its first).
        // When the reducer is c_first its own partial, first in the order, is still in v (0 + v == v,
        // so both paths produce the same bits)
        const int cc0 = own_in_regs ? c_first + 1 : c_first;
        if (!own_in_regs) {
#pragma unroll
          for (int m = 0; m < MP; ++m) v[m] = 0.f;
        }
        // slots per batch of loads: each batch is one L2 round trip (1-3 us while the weight stream
        // loads the L2), so as many as the registers allow (out-proj at b32 has 5-6 contributors)
        constexpr int SL = MP >= 64 ? 2 : (MP >= 32 ? 5 : 8);
        for (int cc = cc0; cc <= c_last; cc += SL) {
          float a[SL][MP];
#pragma unroll
          for (int t = 0; t < SL; ++t) {
            const int c2 = cc + t;
            const float* sl = p.ws + (2LL * c2 + (c2 == c_first && U * c2 / G < t0 ? 1 : 0)) * MP * kBM + col;
#pragma unroll
            for (int m = 0; m < MP; ++m) a[t][m] = c2 <= c_last ? __ldcg(sl + m * kBM) : 0.f;
          }
#pragma unroll
          for (int t = 0; t < SL; ++t)
#pragma unroll
            for (int m = 0; m < MP; ++m)
              if (cc + t <= c_last) v[m] += a[t][m];
        }
        if (threadIdx.x == 128) gstamp(6);
      }
      if (n < p.N) {
        const float bias = p.bias != nullptr ? __half2float(p.bias[n]) : 0.f;
        const bool scaled = n < p.scale_cols;
        const int seg = n / p.seg_width;
        const int scol = n - seg * p.seg_width;
        char* sp = static_cast<char*>(seg == 0 ? p.seg_ptr[0] : (seg == 1 ? p.seg_ptr[1] : p.seg_ptr[2]));
        const long long gs = seg == 0 ? p.seg_group_stride[0] : (seg == 1 ? p.seg_group_stride[1] : p.seg_group_stride[2]);
        const bool f32 = (p.flags & KVPR_EPI_F32) != 0, accum = f32 && (p.flags & KVPR_EPI_ACCUM);
        // residual add: every old value is loaded before the first store -- interleaved
        // load / store pairs would be serialised (possible aliasing), one L2 round trip per row
        const long long ld = p.ld;
        const int rg = p.row_group;
        // (MP = 64 keeps the interleaved form: 64 more live registers would spill)
        constexpr int HOIST = MP <= 32 ? MP : 1;
        auto store_rows = [&](auto off_of) {
          float old[HOIST];
          if constexpr (MP <= 32) {
#pragma unroll
            for (int m = 0; m < MP; ++m)
              old[m] = (accum && m < p.M) ? reinterpret_cast<const float*>(sp)[off_of(m)] : 0.f;
          }
#pragma unroll
          for (int m = 0; m < MP; ++m) {
            if (m >= p.M) continue;
            float x = v[m] + bias;
            if (scaled) x *= p.scale;
            if (p.flags & KVPR_EPI_RELU) x = fmaxf(x, 0.f);
            if (f32) {
              float* o = reinterpret_cast<float*>(sp) + off_of(m);
              if constexpr (MP <= 32) *o = accum ? old[m] + x : x;
              else *o = accum ? *o + x : x;
            } else {
              reinterpret_cast<__half*>(sp)[off_of(m)] = __float2half_rn(x);
            }
          }
        };
        if (rg >= MP)  // one row group (every decode GEMM): a plain stride, no division per row
          store_rows([&](int m) { return static_cast<long long>(m) * ld + scol; });
        else
          store_rows([&](int m) { return static_cast<long long>(m % rg) * ld + static_cast<long long>(m / rg) * gs + scol; });
        if (threadIdx.x == 128) gstamp(7);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) gstamp(5);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// host side

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) != cudaSuccess ||
        qres != cudaDriverEntryPointSuccess) {
      return nullptr;
    }
    fn = reinterpret_cast<PFN_encodeTiled_t>(ptr);
  }
  return fn;
}

// Row-major fp16 matrix [rows, cols] with row stride ld (elements) -> K-major 128B-swizzled boxes.
static int make_tmap(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (enc == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return KVPR_ECUDA;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%llu cols=%llu ld=%llu", int(r),
              (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)ld);
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}

// fp16 tensor [dims[rank-1]]...[dims[0]] with byte strides of dims 1.. (strides[rank-1]) -> boxes `box`
// with the 128-byte swizzle, zero fill out of bounds (prefill_attn.cu's 3-D views of the page layout)
int make_tmap_nd(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                 const uint32_t* box) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (enc == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return KVPR_ECUDA;
  }
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], estr[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    estr[i] = 1;
    if (i + 1 < rank) st[i] = strides[i];
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank, const_cast<void*>(ptr), d, st, bx, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for a rank-%d map", int(r), rank);
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}

// 64-wide k-boxes per ring stage of the swap-AB decode GEMM: KVPR_SWAP_KBOX = 1, 2 or 4 overrides
// the shape-based default (0)
static int swap_kbox() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KVPR_SWAP_KBOX");
    v = (e != nullptr && (atoi(e) == 1 || atoi(e) == 2 || atoi(e) == 4)) ? atoi(e) : 0;
  }
  return v;
}

// Rasterization band (tile_coords): +g = bands of g m-blocks (B re-read once per band), -g =
// bands of g n-blocks (A re-read once per band); whichever reads less from DRAM.  blk_bytes is
// one m-block of A = one n-block of B (both rows x K fp16 for square tiles).
static int band_group(int num_m_blk, int num_n_blk, long long a_blk_bytes, long long b_blk_bytes) {
  static int forced = -1000000;  // experiment override KVPR_GEMM_GROUP_M (negative: n-bands), read once
  if (forced == -1000000) {
    const char* e = getenv("KVPR_GEMM_GROUP_M");
    forced = e != nullptr ? atoi(e) : 0;
  }
  if (forced != 0) return forced;
  long long gm = kABandBytes / (a_blk_bytes > 0 ? a_blk_bytes : 1);
  long long gn = kABandBytes / (b_blk_bytes > 0 ? b_blk_bytes : 1);
  gm = gm < 1 ? 1 : (gm > num_m_blk ? num_m_blk : gm);
  gn = gn < 1 ? 1 : (gn > num_n_blk ? num_n_blk : gn);
  const long long a_all = a_blk_bytes * num_m_blk, b_all = b_blk_bytes * num_n_blk;
  const long long reads_m = a_all + b_all * ((num_m_blk + gm - 1) / gm);
  const long long reads_n = b_all + a_all * ((num_n_blk + gn - 1) / gn);
  return reads_n < reads_m ? -static_cast<int>(gn) : static_cast<int>(gm);
}

template <int BN>
static int launch_bn(const void* a, long long lda, const void* w, long long ldw, GemmArgs args, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ta, tb;
  args.a_box_rows = args.M < kBM ? ((args.M + 7) / 8) * 8 : kBM;
  int rc = make_tmap(&ta, a, args.M, args.K, lda, args.a_box_rows);
  if (rc) return rc;
  rc = make_tmap(&tb, w, args.N, args.K, ldw, BN);
  if (rc) return rc;
  args.num_m_blk = (args.M + kBM - 1) / kBM;
  args.num_n_blk = (args.N + BN - 1) / BN;
  args.num_k_blk = (args.K + kBK - 1) / kBK;
  args.group_m = band_group(args.num_m_blk, args.num_n_blk, static_cast<long long>(kBM) * args.K * 2,
                            static_cast<long long>(BN) * args.K * 2);
  const int splits = args.k_splits > 1 ? args.k_splits : 1;
  const int tiles = args.num_m_blk * args.num_n_blk * splits;
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_done[64] = {0};
  if (dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(gemm_tcgen05_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    attr_done[dev] = 1;
  }
  int grid = tiles < sm_count(dev) ? tiles : sm_count(dev);
  if (args.max_ctas > 0 && grid > args.max_ctas) grid = args.max_ctas;
  int rc2 = launch("gemm_tcgen05", gemm_tcgen05_kernel<BN>, grid, 256, Cfg::kSmemBytes, stream, ta, tb, args);
  if (rc2 || splits == 1) return rc2;
  const long long work = static_cast<long long>(args.M) * (args.N / 32);
  return launch("split_k_reduce", split_k_reduce_kernel, static_cast<unsigned>((work + 127) / 128), 128, 0, stream,
                args);
}


template <int MP, int KB>
static int launch_swapab(const void* a, long long lda, const void* w, long long ldw, GemmArgs args,
                         cudaStream_t stream) {
  using Cfg = SwapCfg<MP, KB>;
  CUtensorMap tw, tx;
  const long long tiled_rows = static_cast<long long>((args.N + kBM - 1) / kBM) * ((args.K + kBK - 1) / kBK) * kBM;
  int rc = args.w_tiled ? make_tmap(&tw, w, tiled_rows, kBK, kBK, kBM) : make_tmap(&tw, w, args.N, args.K, ldw, kBM);
  if (rc) return rc;
  rc = make_tmap(&tx, a, args.M, args.K, lda, MP);  // rows >= M of the box are zero-filled
  if (rc) return rc;
  args.num_m_blk = 1;
  args.num_n_blk = (args.N + kBM - 1) / kBM;
  args.num_k_blk = (args.K + kBK - 1) / kBK;
  args.a_box_rows = MP;
  args.k_splits = 1;
  int dev = 0;
  cudaGetDevice(&dev);
  constexpr uint32_t smem = 1024 + Cfg::kStages * Cfg::kStageBytes + kBarrierBytes;
  static int attr_done[64] = {0};
  if (dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(gemm_swapab_kernel<MP, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_done[dev] = 1;
  }
  // stream-K: one CTA per SM over equal unit ranges; otherwise whole tiles, grid-strided
  const int grid = args.sk_ctas > 0 ? args.sk_ctas : (args.num_n_blk < sm_count(dev) ? args.num_n_blk : sm_count(dev));
  return launch("gemm_swapab", gemm_swapab_kernel<MP, KB>, grid, 256, smem, stream, tw, tx, args);
}

static int launch_2sm(const void* a, long long lda, const void* w, long long ldw, GemmArgs args, cudaStream_t stream) {
  CUtensorMap ta, tb;
  int rc = make_tmap(&ta, a, args.M, args.K, lda, kBM);
  if (rc) return rc;
  rc = make_tmap(&tb, w, args.N, args.K, ldw, k2BN / 2);
  if (rc) return rc;
  args.num_m_blk = (args.M + 2 * kBM - 1) / (2 * kBM);
  args.num_n_blk = (args.N + k2BN - 1) / k2BN;
  args.num_k_blk = (args.K + kBK - 1) / kBK;
  args.group_m = band_group(args.num_m_blk, args.num_n_blk, static_cast<long long>(2 * kBM) * args.K * 2,
                            static_cast<long long>(k2BN) * args.K * 2);
  const int tiles = args.num_m_blk * args.num_n_blk;
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_done[64] = {0};
  if (dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(gemm_tcgen05_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, k2SmemBytes);
    attr_done[dev] = 1;
  }
  int pairs = sm_count(dev) / 2;
  if (args.max_ctas > 1 && pairs > args.max_ctas / 2) pairs = args.max_ctas / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);
  return launch("gemm_tcgen05_2sm", gemm_tcgen05_2sm_kernel, grid, 256, k2SmemBytes, stream, ta, tb, args);
}

// Stream-K arrival counters: one zeroed block of kSkMaxTiles counters per (device, stream), made on first
// use.  Launches on one stream are ordered (the epilogue waits for the previous grid before touching
// them) and the last arrival of every tile returns its counter to zero, so a block is reusable by the
// next call; distinct streams get distinct blocks, so concurrent GEMMs never share one.
static unsigned* sk_counters_for(int dev, cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, unsigned*> blocks;
  std::lock_guard<std::mutex> lock(mu);
  auto it = blocks.find({dev, stream});
  if (it != blocks.end()) return it->second;
  unsigned* p = nullptr;
  if (cudaMalloc(&p, kSkMaxTiles * sizeof(unsigned)) != cudaSuccess ||
      cudaMemsetAsync(p, 0, kSkMaxTiles * sizeof(unsigned), stream) != cudaSuccess) {
    set_error("stream-K counters: device allocation failed");
    return nullptr;
  }
  blocks[{dev, stream}] = p;
  return p;
}

extern "C" int kvpr_debug_gemm_trace(void* buf) {  // tools/sk_trace.py: 8 u64 stamps per CTA, NULL = off
  return cudaMemcpyToSymbol(g_gemm_trace, &buf, sizeof(buf)) == cudaSuccess ? KVPR_OK : KVPR_ECUDA;
}

int gemm_f16(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K, const GemmArgs& epi,
             int bn, cudaStream_t stream, float* ws, size_t ws_bytes, const GemvLn* ln) {
  if (ln != nullptr && bn != kBnGemv) {
    set_error("gemm: a LayerNorm prologue needs the CUDA-core decode projection (bn=-2)");
    return KVPR_EINVAL;
  }
  GemmArgs args = epi;
  args.M = M;
  args.N = N;
  args.K = K;
  args.w_tiled = (epi.flags & KVPR_EPI_W_TILED) ? 1 : 0;
  if (args.w_tiled) {  // only the swap-AB decode GEMM reads the box-tiled layout
    if (M > 64 || (bn != 0 && bn != kBnSwapAB)) {
      set_error("gemm: tiled weights (KVPR_EPI_W_TILED) need the swap-AB decode GEMM (M <= 64, bn 0 or -1)");
      return KVPR_EINVAL;
    }
    bn = kBnSwapAB;
  }
  args.k_splits = 1;
  args.ws = nullptr;
  args.ws_ld = N;
  args.sk_ctas = 0;
  args.sk_counters = nullptr;
  if (bn == kBnSwapAB && ws != nullptr && M > 0 && M <= 64 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0) {
    // weight-streaming decode GEMM: HBM needs every SM streaming for the whole kernel, so stream-K
    // spreads the n-tile x k-block units evenly over all SMs (KVPR_STREAMK=0: whole tiles instead)
    static const bool sk_on = [] {
      const char* e = getenv("KVPR_STREAMK");
      return !(e != nullptr && e[0] == '0');
    }();
    int dev = 0;
    cudaGetDevice(&dev);
    const long long n_tiles = (N + kBM - 1) / kBM;
    const long long units = n_tiles * ((K + kBK - 1) / kBK);
    const int G = static_cast<int>(units < sm_count(dev) ? units : sm_count(dev));
    const int mp = M <= 16 ? 16 : (M <= 32 ? 32 : 64);
    const size_t slots = 2ull * G * mp * kBM * sizeof(float);
    // whole tiles already cover >= 3/4 of the SMs (fc1, LM head): stream-K's fixup costs more than
    // the idle SMs (tools/decode_gemm_tiled.py: fc1 28.9 us whole tiles vs 35.6 stream-K)
    const bool sparse = n_tiles * 4 < 3LL * sm_count(dev);
    if (sk_on && sparse && n_tiles <= kSkMaxTiles && slots <= ws_bytes) {
      unsigned* ctr = sk_counters_for(dev, stream);
      if (ctr == nullptr) return KVPR_ECUDA;
      args.sk_ctas = G;
      args.ws = ws;
      args.sk_counters = ctr;
    }
  } else if (ws != nullptr && M <= kBM && bn > 0 && bn <= 256 && K >= 8192) {
    // only long k-loops gain: short ones are dominated by pipeline fill + the extra reduce launch
    // (measured: fc2 32x4096x16384 75 -> 51 us; out-proj 32x4096x4096 23 -> 29 us)
    // one row block, weight-streaming: each CTA's k-loop is latency bound, so slice K until the
    // CTAs fill the SMs (deterministic: partials reduced in slice order by a second kernel)
    int dev = 0;
    cudaGetDevice(&dev);
    const int n_tiles = (N + bn - 1) / bn;
    const int num_kb = (K + kBK - 1) / kBK;
    int s = sm_count(dev) / n_tiles;
    if (s > 8) s = 8;
    while (s > 1 && (num_kb + s - 1) / s * (s - 1) >= num_kb) --s;  // every slice non-empty
    if (s > 1 && static_cast<size_t>(s) * M * N * sizeof(float) <= ws_bytes &&
        (reinterpret_cast<uintptr_t>(ws) & 15) == 0) {
      args.k_splits = s;
      args.ws = ws;
    }
  }
  if (M <= 0 || N <= 0 || K <= 0) {
    set_error("gemm: non-positive shape M=%d N=%d K=%d", M, N, K);
    return KVPR_EINVAL;
  }
  if (N % 32 != 0 || K % 8 != 0 || lda % 8 != 0 || (!args.w_tiled && ldw % 8 != 0)) {
    set_error("gemm: need N%%32==0, K%%8==0, lda/ldw%%8==0 (N=%d K=%d lda=%lld ldw=%lld)", N, K, lda, ldw);
    return KVPR_EINVAL;
  }
  if ((reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(w) & 15)) {
    set_error("gemm: operands must be 16-byte aligned");
    return KVPR_EINVAL;
  }
  if (args.seg_width <= 0 || args.seg_width % 32 != 0 || args.row_group <= 0) {
    set_error("gemm: epilogue seg_width must be a positive multiple of 32 and row_group > 0");
    return KVPR_EINVAL;
  }
  const int nseg = (N + args.seg_width - 1) / args.seg_width;
  if (nseg > 3) {
    set_error("gemm: at most 3 output segments (N=%d seg_width=%d)", N, args.seg_width);
    return KVPR_EINVAL;
  }
  for (int s = 0; s < nseg; ++s) {
    if (args.seg_ptr[s] == nullptr || (reinterpret_cast<uintptr_t>(args.seg_ptr[s]) & 15)) {
      set_error("gemm: output segment %d pointer null or misaligned", s);
      return KVPR_EINVAL;
    }
  }
  if (args.bias != nullptr && (reinterpret_cast<uintptr_t>(args.bias) & 15)) {
    set_error("gemm: bias must be 16-byte aligned");
    return KVPR_EINVAL;
  }
  switch (bn) {
    case kBnGemv:
      return gemv_f16(a, lda, w, ldw, args, stream, ln);
    case kBnSwapAB:  // weight-streaming decode GEMM, M <= 64
      if (M > 64) {
        set_error("gemm: swap-AB decode GEMM needs M <= 64 (M=%d)", M);
        return KVPR_EINVAL;
      }
      {
        // measured (tools/decode_gemm_bench.py --swap-only, KVPR_SWAP_KBOX): 4 boxes per stage at
        // M <= 16, 2 above (larger stages, fewer of them, once the activation box grows)
        const int kb = swap_kbox() > 0 ? swap_kbox() : (M <= 16 ? 4 : 2);
        if (M <= 16) return kb == 4 ? launch_swapab<16, 4>(a, lda, w, ldw, args, stream)
                                    : (kb == 2 ? launch_swapab<16, 2>(a, lda, w, ldw, args, stream)
                                               : launch_swapab<16, 1>(a, lda, w, ldw, args, stream));
        if (M <= 32) return kb == 4 ? launch_swapab<32, 4>(a, lda, w, ldw, args, stream)
                                    : (kb == 2 ? launch_swapab<32, 2>(a, lda, w, ldw, args, stream)
                                               : launch_swapab<32, 1>(a, lda, w, ldw, args, stream));
        return kb == 4 ? launch_swapab<64, 4>(a, lda, w, ldw, args, stream)
                       : (kb == 2 ? launch_swapab<64, 2>(a, lda, w, ldw, args, stream)
                                  : launch_swapab<64, 1>(a, lda, w, ldw, args, stream));
      }
    case 512:  // 256 x 256 pair tile on a CTA pair (cta_group::2)
      return launch_2sm(a, lda, w, ldw, args, stream);
    case 256:
      return launch_bn<256>(a, lda, w, ldw, args, stream);
    case 128:
      return launch_bn<128>(a, lda, w, ldw, args, stream);
    case 64:
      return launch_bn<64>(a, lda, w, ldw, args, stream);
    case 32:  // small-M weight streaming with few output columns: more CTAs in flight
      return launch_bn<32>(a, lda, w, ldw, args, stream);
    default:
      set_error("gemm: unsupported BN=%d", bn);
      return KVPR_EINVAL;
  }
}

}  // namespace kvpr

namespace kvpr {

// W [N, K] row-major (row stride ldw) -> box-tiled [n_blk][k_blk][128][64], zero-padded to whole boxes:
// the layout the swap-AB decode GEMM streams as contiguous 16 KB boxes (KVPR_EPI_W_TILED).  One
// thread per 8 consecutive k (16 bytes).
__global__ void tile_weight_kernel(const __half* __restrict__ w, long long ldw, int N, int K, int nkb,
                                   __half* __restrict__ out, long long total_vec) {
  const long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= total_vec) return;
  const long long e = v * 8;                 // element index in the tiled buffer
  const int c = static_cast<int>(e % kBK);   // k inside the box
  const long long rowt = e / kBK;            // row of the [*, 64] view
  const int r = static_cast<int>(rowt % kBM);
  const long long box = rowt / kBM;
  const int kb = static_cast<int>(box % nkb);
  const long long nb = box / nkb;
  const long long n = nb * kBM + r;
  const int k = kb * kBK + c;
  uint4 val = make_uint4(0, 0, 0, 0);
  if (n < N && k + 8 <= K) val = *reinterpret_cast<const uint4*>(w + n * ldw + k);
  else if (n < N) {
    __half h[8];
    for (int i = 0; i < 8; ++i) h[i] = k + i < K ? w[n * ldw + k + i] : __float2half(0.f);
    val = *reinterpret_cast<uint4*>(h);
  }
  *reinterpret_cast<uint4*>(out + e) = val;
}

size_t tiled_weight_bytes(int N, int K) {
  if (N <= 0 || K <= 0) return 0;
  return static_cast<size_t>((N + kBM - 1) / kBM) * ((K + kBK - 1) / kBK) * kBM * kBK * sizeof(__half);
}

int tile_weight(const void* w, long long ldw, int N, int K, void* out, cudaStream_t stream) {
  if (w == nullptr || out == nullptr || N <= 0 || K <= 0 || ldw < K || (reinterpret_cast<uintptr_t>(w) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15) || ldw % 8 != 0) {
    set_error("tile_weight: need non-null 16-byte aligned w / out, N, K > 0, ldw >= K, ldw %% 8 == 0");
    return KVPR_EINVAL;
  }
  const int nkb = (K + kBK - 1) / kBK;
  const long long total_vec = static_cast<long long>(tiled_weight_bytes(N, K) / 16);
  return launch("tile_weight", tile_weight_kernel, static_cast<unsigned>((total_vec + 255) / 256), 256, 0, stream,
                static_cast<const __half*>(w), ldw, N, K, nkb, static_cast<__half*>(out), total_vec);
}

// Push half of the fused TP all-reduce: the swap-AB decode GEMM whose epilogue stores raw fp32
// partials into the tile owners' receive slots and releases their flags (csrc/tpcomm.cu).
int gemm_tp_partials(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                     const GemmArgs& tp, cudaStream_t stream) {
  if (M <= 0 || M > 64 || N <= 0 || K <= 0 || N % 32 != 0 || K % 8 != 0 || lda % 8 != 0 || ldw % 8 != 0) {
    set_error("linear_allreduce: need 0 < M <= 64, N %% 32 == 0, K %% 8 == 0 (M=%d N=%d K=%d)", M, N, K);
    return KVPR_EINVAL;
  }
  if ((N + kBM - 1) / kBM > kTpMaxTiles) {
    set_error("linear_allreduce: N=%d exceeds %d tiles of %d", N, kTpMaxTiles, kBM);
    return KVPR_EINVAL;
  }
  GemmArgs args = tp;
  args.M = M;
  args.N = N;
  args.K = K;
  args.k_splits = 1;
  args.ws = nullptr;
  args.seg_width = ((N + 31) / 32) * 32;
  args.row_group = M;
  const int kb = swap_kbox() > 0 ? swap_kbox() : (M <= 16 ? 4 : 2);
  if (M <= 16) return kb == 4 ? launch_swapab<16, 4>(a, lda, w, ldw, args, stream)
                              : launch_swapab<16, 2>(a, lda, w, ldw, args, stream);
  if (M <= 32) return kb == 4 ? launch_swapab<32, 4>(a, lda, w, ldw, args, stream)
                              : launch_swapab<32, 2>(a, lda, w, ldw, args, stream);
  return kb == 4 ? launch_swapab<64, 4>(a, lda, w, ldw, args, stream)
                 : launch_swapab<64, 2>(a, lda, w, ldw, args, stream);
}

}  // namespace kvpr
