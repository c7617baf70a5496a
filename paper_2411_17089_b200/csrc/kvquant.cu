// 4-bit groupwise KV pages: the cache that crosses PCIe
// is stored at kv_bytes_per_element = 0.5625 = 4/8 + 4/64, i.e. 4-bit codes in
// groups of 64 along the hidden dimension with an fp16 (min, scale) pair per
// group — costmodel.groupwise_quant_bytes_per_element(4, 64, 4)
// (costmodel.py:109-118), asymmetric min/max quantisation as in FlexGen.
//
// Compressed page (one position, whole batch, K then V), contiguous so a
// position range is one DMA:
//   codes  : [2][batch][hidden/2] bytes  (element 2i in the low nibble, 2i+1 high)
//   params : [2][batch][hidden/64][2] fp16 (min, scale)
// page bytes = 2*batch*hidden*0.5625.
//
// Arithmetic (bit-exact with oracle/opt_ref.py's emulation):
//   mn = half(min g), sc = half((max g - float(mn)) / 15)
//   q  = clamp(rint((x - mn) / sc), 0, 15)   (q = 0 when sc == 0)
//   x^ = half(mn + q * sc)                   (no FMA contraction)
// One warp per group of 64: each lane owns two elements (one code byte).

#include <stdlib.h>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {

namespace {

__global__ void kv4_quantize_kernel(const __half* __restrict__ pages, uint8_t* __restrict__ qpages, int batch,
                                    int hidden, int pos_begin, long long groups_per_page, long long total_groups) {
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= total_groups) return;
  const long long p = pos_begin + gw / groups_per_page;
  const long long g = gw % groups_per_page;  // group within the page: ((kv*batch + b) * hidden/64 + j)
  const long long page_elems = 2LL * batch * hidden;
  const long long page_bytes = page_elems / 2 + (page_elems / 64) * 4;
  const __half2 x2 = reinterpret_cast<const __half2*>(pages + p * page_elems + g * 64)[lane];
  const float2 x = __half22float2(x2);
  float mn = fminf(x.x, x.y), mx = fmaxf(x.x, x.y);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const __half mn16 = __float2half_rn(mn);
  const float mnf = __half2float(mn16);
  const __half sc16 = __float2half_rn(__fdiv_rn(__fsub_rn(mx, mnf), 15.f));
  const float sc = __half2float(sc16);
  int q0 = 0, q1 = 0;
  if (sc > 0.f) {
    q0 = static_cast<int>(rintf(__fdiv_rn(__fsub_rn(x.x, mnf), sc)));
    q1 = static_cast<int>(rintf(__fdiv_rn(__fsub_rn(x.y, mnf), sc)));
    q0 = min(max(q0, 0), 15);
    q1 = min(max(q1, 0), 15);
  }
  uint8_t* qp = qpages + p * page_bytes;
  qp[g * 32 + lane] = static_cast<uint8_t>(q0 | (q1 << 4));
  if (lane == 0) {
    __half2 prm = __halves2half2(mn16, sc16);
    reinterpret_cast<__half2*>(qp + page_elems / 2)[g] = prm;
  }
}

__global__ void kv4_dequantize_kernel(const uint8_t* __restrict__ qpages, __half* __restrict__ pages, int batch,
                                      int hidden, int pos_begin, long long groups_per_page, long long total_groups) {
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= total_groups) return;
  const long long p = pos_begin + gw / groups_per_page;
  const long long g = gw % groups_per_page;
  const long long page_elems = 2LL * batch * hidden;
  const long long page_bytes = page_elems / 2 + (page_elems / 64) * 4;
  const uint8_t* qp = qpages + p * page_bytes;
  const uint8_t code = qp[g * 32 + lane];
  const float2 prm = __half22float2(reinterpret_cast<const __half2*>(qp + page_elems / 2)[g]);
  const float a = __fadd_rn(prm.x, __fmul_rn(static_cast<float>(code & 15), prm.y));
  const float b = __fadd_rn(prm.x, __fmul_rn(static_cast<float>(code >> 4), prm.y));
  reinterpret_cast<__half2*>(pages + p * page_elems + g * 64)[lane] = __floats2half2_rn(a, b);
}

int kv4_check(int batch, int hidden, int pos_begin, int pos_end, const void* a, const void* b) {
  if (batch <= 0 || hidden <= 0 || hidden % 64 != 0 || pos_begin < 0 || pos_end < pos_begin) {
    set_error("kv4: need batch > 0, hidden %% 64 == 0, 0 <= pos_begin <= pos_end (got b=%d h=%d [%d,%d))", batch,
              hidden, pos_begin, pos_end);
    return KVPR_EINVAL;
  }
  if (pos_end > pos_begin && (a == nullptr || b == nullptr)) {
    set_error("kv4: null pointer");
    return KVPR_EINVAL;
  }
  return KVPR_OK;
}

}  // namespace

size_t kv4_page_bytes(int batch, int hidden) {
  const size_t e = 2ull * batch * hidden;
  return e / 2 + (e / 64) * 4;
}

int kv4_quantize(const __half* pages, uint8_t* qpages, int batch, int hidden, int pos_begin, int pos_end,
                 cudaStream_t stream) {
  int rc = kv4_check(batch, hidden, pos_begin, pos_end, pages, qpages);
  if (rc || pos_end == pos_begin) return rc;
  const long long gpp = 2LL * batch * hidden / 64;
  const long long total = gpp * (pos_end - pos_begin);
  const int threads = 256;
  const long long blocks = (total * 32 + threads - 1) / threads;
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  kv4_quantize_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(pages, qpages, batch, hidden, pos_begin,
                                                                             gpp, total);
  return check_launch("kv4_quantize");
}

int kv4_dequantize(const uint8_t* qpages, __half* pages, int batch, int hidden, int pos_begin, int pos_end,
                   cudaStream_t stream) {
  int rc = kv4_check(batch, hidden, pos_begin, pos_end, qpages, pages);
  if (rc || pos_end == pos_begin) return rc;
  const long long gpp = 2LL * batch * hidden / 64;
  const long long total = gpp * (pos_end - pos_begin);
  const int threads = 256;
  const long long blocks = (total * 32 + threads - 1) / threads;
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  kv4_dequantize_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(qpages, pages, batch, hidden,
                                                                               pos_begin, gpp, total);
  return check_launch("kv4_dequantize");
}

}  // namespace kvpr

// ---------------------------------------------------------------------------
// Diagnostic: host -> device copy driven by SM loads from page-locked host memory (UVA,
// zero-copy) instead of a copy engine.  Used by tools/k2_probe.py to tell copy-engine/PCIe-write
// interference apart from PCIe-read traffic; not on the decode path.
namespace kvpr {
namespace {
template <int U>
__global__ void __launch_bounds__(1024) sm_pull_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                       long long n16) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * U;
  for (long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * U; i < n16; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u < n16) v[u] = src[i + u];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u < n16) dst[i + u] = v[u];
  }
}
}  // namespace
}  // namespace kvpr

// threads per CTA and 16-byte loads in flight per thread come from KVPR_PULL_THREADS (256) and
// KVPR_PULL_UNROLL (4 / 8 / 16; default 4): bytes in flight per SM = threads x unroll x 16
extern "C" int kvpr_debug_sm_pull(const void* host, void* dev, size_t bytes, int ctas, void* stream) {
  using namespace kvpr;
  if (host == nullptr || dev == nullptr || bytes % 16 != 0 || ctas <= 0) {
    set_error("debug_sm_pull: need non-null pointers, bytes %% 16 == 0, ctas > 0");
    return KVPR_EINVAL;
  }
  const char* te = getenv("KVPR_PULL_THREADS");
  const char* ue = getenv("KVPR_PULL_UNROLL");
  const int threads = te != nullptr && atoi(te) >= 32 && atoi(te) <= 1024 ? atoi(te) : 256;
  const int unroll = ue != nullptr ? atoi(ue) : 4;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint4* src = static_cast<const uint4*>(host);
  uint4* dst = static_cast<uint4*>(dev);
  const long long n16 = static_cast<long long>(bytes / 16);
  if (unroll >= 16)
    sm_pull_kernel<16><<<ctas, threads, 0, s>>>(src, dst, n16);
  else if (unroll >= 8)
    sm_pull_kernel<8><<<ctas, threads, 0, s>>>(src, dst, n16);
  else
    sm_pull_kernel<4><<<ctas, threads, 0, s>>>(src, dst, n16);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return check_launch("debug_sm_pull");
}
