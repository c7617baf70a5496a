// Decode-attention building blocks shared by K2 (attention.cu) and the fused small-batch layer
// tail (layer_tail.cu): 16-byte K/V loads, the exp2-domain online softmax of one lane group, the
// position sweep and the in-warp merge.  One definition, so both kernels sweep with the same
// arithmetic.  Reference semantics: numerics.decode_attention / stable_softmax (numerics.py:159-191).
#pragma once

#include <math.h>

#include "common.cuh"

namespace kvpr {
namespace attn {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void load8(const __half* p, float (&f)[8]) {
  uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __half22float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Streamed (read-once) variant for the big K/V sweep: bypass L1 allocation.
__device__ __forceinline__ uint4 ld_stream(const __half* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __half22float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Online-softmax state of one lane group: running max (log2 domain), sum, acc[8].
struct Softmax8 {
  float m, l, acc[8];
  __device__ __forceinline__ void init() {
    m = -INFINITY;
    l = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  }
};

// Sweep positions p = first, first+step, ... < end with a group of LPP lanes
// per position, U positions in flight per lane.  q8 is pre-multiplied by
// scale*log2e so scores come out in the exp2 domain.
// `first` must be warp-uniform (the shuffles below need the whole warp in every
// trip); lane group `grp` owns positions first + grp + u*step + trip*U*step.
// Positions [lo, hi) of the sweep read 4-bit compressed pages (kvquant.cu layout) instead of the
// fp16 page buffer: the transferred tail of the kv_bits=4 path, dequantised in registers with the
// exact arithmetic of kv4_dequantize_kernel (x^ = half(min + q*scale), no FMA), so K2 sees the
// same fp16 values as after a separate dequantize pass — without writing and re-reading them.
struct Q4Src {
  const uint8_t* base;  // compressed page of position 0
  long long page_bytes;
  long long ck, cv, pk, pv;  // this lane's K/V code and (min, scale) byte offsets within a page
  int lo, hi;
};

__device__ __forceinline__ uint32_t ld_stream32(const uint8_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 deq8(uint32_t codes, uint32_t prm) {
  __half2 mp = *reinterpret_cast<const __half2*>(&prm);
  const float2 f = __half22float2(mp);
  uint4 out;
  uint32_t* o = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t byte = (codes >> (8 * i)) & 0xffu;
    const float a = __fadd_rn(f.x, __fmul_rn(static_cast<float>(byte & 15u), f.y));
    const float b = __fadd_rn(f.x, __fmul_rn(static_cast<float>(byte >> 4), f.y));
    __half2 h = __floats2half2_rn(a, b);
    o[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return out;
}

// Positions [lo, hi) read from `base` instead, position p's K at base + (p - lo) * stride (+ the lane's
// 8 elements), its V v_off further, with generic loads (global, mapped host or shared memory): the fused
// layer tail's copy of the transferred tail KV[l:s'-1], pulled from the host store into shared memory.
struct AltSrc {
  const __half* base;
  int lo, hi;
  int stride, v_off;
};

template <int D, int U, bool Q4 = false, bool ALT = false>
__device__ __forceinline__ void sweep(const __half* __restrict__ kbase, long long page_stride, long long v_off,
                                      int first, int end, int step, int grp, const float (&q8)[8], int glane,
                                      Softmax8& st, const Q4Src* qs = nullptr, const AltSrc* alt = nullptr) {
  constexpr int LPP = D / 8;
  for (int pb = first; pb < end; pb += step * U) {
    const int p0 = pb + grp;
    uint4 kr[U], vr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = p0 + u * step;
      kr[u] = make_uint4(0, 0, 0, 0);
      vr[u] = make_uint4(0, 0, 0, 0);
      if (p < end) {
        if (Q4 && p >= qs->lo && p < qs->hi) {
          const uint8_t* pg = qs->base + (long long)p * qs->page_bytes;
          kr[u] = deq8(ld_stream32(pg + qs->ck), __ldg(reinterpret_cast<const unsigned int*>(pg + qs->pk)));
          vr[u] = deq8(ld_stream32(pg + qs->cv), __ldg(reinterpret_cast<const unsigned int*>(pg + qs->pv)));
        } else if (ALT && p >= alt->lo && p < alt->hi) {
          const __half* kp = alt->base + (p - alt->lo) * alt->stride + glane * 8;
          kr[u] = *reinterpret_cast<const uint4*>(kp);
          vr[u] = *reinterpret_cast<const uint4*>(kp + alt->v_off);
        } else {
          const __half* kp = kbase + (long long)p * page_stride + glane * 8;
          kr[u] = ld_stream(kp);
          vr[u] = ld_stream(kp + v_off);
        }
      }
    }
    float s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float kf[8];
      unpack8(kr[u], kf);
      float d = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) d = fmaf(q8[i], kf[i], d);
#pragma unroll
      for (int o = LPP / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      s[u] = (p0 + u * step < end) ? d : -INFINITY;
    }
    float mx = st.m;
#pragma unroll
    for (int u = 0; u < U; ++u) mx = fmaxf(mx, s[u]);
    if (mx == -INFINITY) continue;  // whole block masked (only possible past `end`)
    const float corr = exp2f(st.m - mx);
    st.l *= corr;
#pragma unroll
    for (int i = 0; i < 8; ++i) st.acc[i] *= corr;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float pw = exp2f(s[u] - mx);
      if (p0 + u * step < end) {
        float vf[8];
        unpack8(vr[u], vf);
        st.l += pw;
#pragma unroll
        for (int i = 0; i < 8; ++i) st.acc[i] = fmaf(pw, vf[i], st.acc[i]);
      }
    }
    st.m = mx;
  }
}

// Merge softmax states of lanes that own the same 8 dims (xor over lane-group index bits).
template <int LPP>
__device__ __forceinline__ void merge_in_warp(Softmax8& st) {
#pragma unroll
  for (int o = LPP; o < 32; o <<= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, st.m, o);
    const float ol = __shfl_xor_sync(0xffffffffu, st.l, o);
    const float nm = fmaxf(st.m, om);
    const float a = (st.m == -INFINITY) ? 0.f : exp2f(st.m - nm);
    const float b = (om == -INFINITY) ? 0.f : exp2f(om - nm);
    st.l = st.l * a + ol * b;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float oa = __shfl_xor_sync(0xffffffffu, st.acc[i], o);
      st.acc[i] = st.acc[i] * a + oa * b;
    }
    st.m = nm;
  }
}

}  // namespace attn
}  // namespace kvpr
