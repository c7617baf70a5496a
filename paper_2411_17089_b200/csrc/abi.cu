// extern "C" boundary of libkvpr.so (declared in include/kvpr.h).
//
// Validation mirrors the reference's ValueError conditions where one exists
// (numerics.py:22-32, 121-126, 172-182); everything else is a CUDA error.
// No entry point allocates, frees or synchronises.

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "kvpr_internal.h"

namespace kvpr {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = 0; }

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}

std::atomic<long long> g_kernel_launches{0};

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KVPR_PDL");
    v = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// KVPR_GEMV: the largest weight (MB) auto mode routes to the CUDA-core decode projection;
// 0 = never, < 0 = any size (A/B knob for tools/decode_gemm_bench.py).  Default 8 MB: below it the
// swap-AB kernel has too few 128-row tiles to stream at HBM rate; above it, it has enough
static long long gemv_max_weight_bytes() {
  static long long v = -2;
  if (v == -2) {
    const char* e = getenv("KVPR_GEMV");
    v = e == nullptr ? (8ll << 20) : static_cast<long long>(atof(e) * (1 << 20));
  }
  return v;
}

int sm_count(int device) {
  static int cache[64] = {0};
  if (device >= 0 && device < 64 && cache[device] > 0) return cache[device];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
  if (device >= 0 && device < 64) cache[device] = n;
  return n;
}

// n DMAs on one stream, one cudaMemcpyAsync each, in order; zero-byte entries dropped.  (The driver's
// batched-copy submission was measured 4 us faster per small layer, tools/dma_small_probe.py, but
// faulted the GPU on this pool, so every copy is its own submission.)
int copy_batch(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t n, cudaStream_t stream) {
  constexpr size_t kMax = 16;
  if (n > kMax) {
    set_error("copy_batch: at most %zu copies per batch (got %zu)", kMax, n);
    return KVPR_EINVAL;
  }
  for (size_t i = 0; i < n; ++i) {
    if (sizes[i] != 0 && (dsts[i] == nullptr || srcs[i] == nullptr)) {
      set_error("copy_batch: null pointer in copy %zu", i);
      return KVPR_EINVAL;
    }
  }
  for (size_t i = 0; i < n; ++i) {
    if (sizes[i] == 0) continue;
    const cudaError_t e = cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDefault, stream);
    if (e != cudaSuccess) {
      set_error("copy_batch: %s", cudaGetErrorString(e));
      return KVPR_ECUDA;
    }
  }
  return KVPR_OK;
}

static GemmArgs to_args(const kvpr_epilogue* e) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.bias = static_cast<const __half*>(e->bias);
  a.seg_width = e->seg_width;
  a.row_group = e->row_group;
  a.ld = e->ld;
  for (int s = 0; s < 3; ++s) {
    a.seg_ptr[s] = e->seg[s].ptr;
    a.seg_group_stride[s] = e->seg[s].group_stride;
  }
  a.scale = e->scale;
  a.scale_cols = e->scale_cols;
  a.flags = e->flags;
  return a;
}

}  // namespace kvpr

using namespace kvpr;

extern "C" {

const char* kvpr_last_error(void) { return g_err; }

int kvpr_version(void) { return 2; }

long long kvpr_kernel_launches(void) { return g_kernel_launches.load(std::memory_order_relaxed); }

int kvpr_sm_count(int device) { return sm_count(device); }

// K1's tile for a launch over `positions` positions: CTA-pair 256x256 tiles (512) when they fill the
// SM pairs; below that (small models, short chunks) the widest 1-CTA tile (BN 32..256) that still
// gives >= sms/2 tiles.  Every shape accumulates K in the same order, so the choice never changes
// a bit (measured: tools/decode_gemm_bench.py --k1-only).  KVPR_K1_BN overrides it (experiments).
int kvpr_recompute_tile(int batch, int positions, int hidden, int sms) {
  if (batch <= 0 || positions <= 0 || hidden <= 0 || sms <= 0) return 0;
  const long long M = static_cast<long long>(positions) * batch;
  const long long N = 2LL * hidden;
  int bn = 512;
  if (((M + 255) / 256) * ((N + 255) / 256) < sms / 2) {
    const long long m_blk = (M + 127) / 128;
    bn = 32;
    for (int c = 256; c >= 32; c /= 2) {
      if (m_blk * ((N + c - 1) / c) >= sms / 2) {
        bn = c;
        break;
      }
    }
  }
  static const int bn_env = [] {
    const char* e = getenv("KVPR_K1_BN");
    const int v = e != nullptr ? atoi(e) : 0;
    return (v == 32 || v == 64 || v == 128 || v == 256 || v == 512) ? v : 0;
  }();
  return bn_env ? bn_env : bn;
}

int kvpr_recompute_kv(const void* x, const void* w_kv, const void* b_kv, void* kv_pages, int batch, int pos_begin,
                      int pos_end, int hidden, void* stream) {
  g_err[0] = 0;
  if (batch <= 0 || hidden <= 0 || pos_begin < 0 || pos_end < pos_begin) {
    set_error("split must satisfy 0 <= pos_begin <= pos_end (got [%d, %d)), batch=%d hidden=%d", pos_begin, pos_end,
              batch, hidden);
    return KVPR_EINVAL;
  }
  if (pos_end == pos_begin) return KVPR_OK;  // split 0: nothing rebuilt (numerics.py:127-128)
  if (x == nullptr || w_kv == nullptr || kv_pages == nullptr) {
    set_error("recompute_kv: null pointer");
    return KVPR_EINVAL;
  }
  const long long bh = (long long)batch * hidden;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.bias = static_cast<const __half*>(b_kv);
  a.seg_width = hidden;                     // columns [0,h) -> K, [h,2h) -> V
  a.row_group = batch;                      // rows of one position
  a.ld = hidden;
  __half* page0 = static_cast<__half*>(kv_pages) + (long long)pos_begin * 2 * bh;
  a.seg_ptr[0] = page0;                     // K half of each page
  a.seg_ptr[1] = page0 + bh;                // V half of each page
  a.seg_group_stride[0] = 2 * bh;           // next position = next page
  a.seg_group_stride[1] = 2 * bh;
  a.scale = 1.f;
  a.scale_cols = 0;
  a.flags = 0;
  const __half* a_ptr = static_cast<const __half*>(x) + (long long)pos_begin * bh;
  const int M = (pos_end - pos_begin) * batch;
  int dev = 0;
  cudaGetDevice(&dev);
  const int bn = kvpr_recompute_tile(batch, pos_end - pos_begin, hidden, sm_count(dev));
  // KVPR_K1_CTAS=n (A/B): K1 on at most n SMs, the rest left to a concurrent layer tail (KVPR_TAIL_CTAS)
  static const int k1_ctas = [] {
    const char* e = getenv("KVPR_K1_CTAS");
    return e != nullptr && atoi(e) > 0 ? atoi(e) : 0;
  }();
  a.max_ctas = k1_ctas;
  return gemm_f16(a_ptr, hidden, w_kv, hidden, M, 2 * hidden, hidden, a, bn, static_cast<cudaStream_t>(stream));
}

int kvpr_linear(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                const kvpr_epilogue* epi, int bn, void* stream) {
  return kvpr_linear_ws(a, lda, w, ldw, M, N, K, epi, bn, nullptr, 0, stream);
}

// bn = 0: the tile / kernel for this shape (has_ws: the caller's entry allows a different k order)
static int auto_bn(int M, int N, int K, bool has_ws) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count(dev);
  const long long m_blk = (M + 127) / 128;
  const long long gemv_cap = gemv_max_weight_bytes();
  if (M <= kGemvMaxM && has_ws && gemv_smem_bytes(M, K) <= static_cast<size_t>(kGemvMaxSmem) &&
      (gemv_cap < 0 || static_cast<long long>(N) * K * 2 <= gemv_cap)) {
    // decode at batch <= 8 through the split-capable entry (out-proj, fc1, fc2, LM head — never
    // the q/k/v projection, whose k, v must carry K1's bits): CUDA-core weight streaming (gemv.cu)
    return -2;
  }
  if (M <= 64) return -1;  // decode (M = batch): weight streaming with the operands swapped (gemm_swapab_kernel)
  if (((M + 255) / 256) * (long long)((N + 255) / 256) >= sms / 2) return 512;
  // one row block: weight-streaming; per-CTA k-loop throughput, not CTA count, limits
  // it, so wide N tiles win (measured: tools/gemm_bench.py, profiles/r01_gemm_variants.jsonl)
  if (m_blk == 1) return 128;
  // large GEMMs: CTA-pair 256x256 tiles when they fill the SM pairs; otherwise narrower N tiles
  // give more CTAs
  int bn = 256;
  if (m_blk * ((N + 255) / 256) < sms) bn = 128;
  if (m_blk * ((N + 127) / 128) < sms) bn = 64;
  return bn;
}

size_t kvpr_tiled_weight_bytes(int N, int K) { return tiled_weight_bytes(N, K); }

int kvpr_tile_weight(const void* w, long long ldw, int N, int K, void* out, void* stream) {
  g_err[0] = 0;
  return tile_weight(w, ldw, N, K, out, static_cast<cudaStream_t>(stream));
}

int kvpr_linear_ws(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                   const kvpr_epilogue* epi, int bn, void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (epi == nullptr || a == nullptr || w == nullptr) {
    set_error("linear: null pointer");
    return KVPR_EINVAL;
  }
  if (bn == 0) bn = (epi->flags & KVPR_EPI_W_TILED) ? -1 : auto_bn(M, N, K, ws != nullptr);
  return gemm_f16(a, lda, w, ldw, M, N, K, to_args(epi), bn, static_cast<cudaStream_t>(stream),
                  static_cast<float*>(ws), ws_bytes);
}

int kvpr_layernorm_linear_ws(const float* x, long long ldx, const void* gamma, const void* beta, float eps, void* y,
                             long long ldy, const void* w, long long ldw, int M, int N, int K,
                             const kvpr_epilogue* epi, int bn, void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (epi == nullptr || x == nullptr || y == nullptr || w == nullptr || gamma == nullptr || beta == nullptr) {
    set_error("layernorm_linear: null pointer");
    return KVPR_EINVAL;
  }
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (bn == 0) bn = (epi->flags & KVPR_EPI_W_TILED) ? -1 : auto_bn(M, N, K, ws != nullptr);
  // KVPR_LN_FUSE=1: the one-launch form.  Off by default: at config 1 it measured 0.736 vs 0.700
  // ms/step with the rows re-read per pass, and 0.7101 vs 0.7067 with the rows held in registers
  // (profiles/r01_ln_fuse_ab.jsonl) — every CTA's LN prologue sits after its PDL wait and costs
  // about what the separate 4-CTA LN launch does
  static const bool fuse = [] {
    const char* e = getenv("KVPR_LN_FUSE");
    return e != nullptr && e[0] == '1';
  }();
  if (bn == -2 && fuse && K <= kGemvLnMaxK) {
    // one launch: every CTA normalises the M rows into its staging buffer (CTA 0 also writes y)
    const GemvLn ln{x, ldx, static_cast<const __half*>(gamma), static_cast<const __half*>(beta), eps,
                    static_cast<__half*>(y), ldy};
    return gemm_f16(y, ldy, w, ldw, M, N, K, to_args(epi), bn, s, static_cast<float*>(ws), ws_bytes, &ln);
  }
  const int rc = layernorm(x, ldx, static_cast<const __half*>(gamma), static_cast<const __half*>(beta),
                           static_cast<__half*>(y), ldy, M, K, eps, s);
  if (rc) return rc;
  return gemm_f16(y, ldy, w, ldw, M, N, K, to_args(epi), bn, s, static_cast<float*>(ws), ws_bytes);
}

int kvpr_decode_attention(const void* q, const void* kv_pages, void* out, void* ws, size_t ws_bytes, int batch,
                          int heads, int head_dim, int seq_len, float scale, void* stream) {
  g_err[0] = 0;
  return decode_attention(static_cast<const __half*>(q), static_cast<const __half*>(kv_pages),
                          static_cast<__half*>(out), static_cast<float*>(ws), ws_bytes, batch, heads, head_dim,
                          seq_len, scale, static_cast<cudaStream_t>(stream));
}

int kvpr_decode_attention_ragged(const void* q, const void* kv_pages, const int* seq_lens, void* out, void* ws,
                                 size_t ws_bytes, int batch, int heads, int head_dim, int max_seq_len, float scale,
                                 void* stream) {
  g_err[0] = 0;
  if (seq_lens == nullptr) {
    set_error("decode_attention_ragged: seq_lens is NULL (use kvpr_decode_attention for a uniform batch)");
    return KVPR_EINVAL;
  }
  return decode_attention(static_cast<const __half*>(q), static_cast<const __half*>(kv_pages),
                          static_cast<__half*>(out), static_cast<float*>(ws), ws_bytes, batch, heads, head_dim,
                          max_seq_len, scale, static_cast<cudaStream_t>(stream), seq_lens);
}

int kvpr_decode_layer_tail_supported(int batch, int hidden, int heads, int ffn) {
  return layer_tail_supported(batch, hidden, heads, ffn) ? 1 : 0;
}

int kvpr_decode_layer_tail(const kvpr_layer_tail_desc* desc, void* stream) {
  g_err[0] = 0;
  if (desc == nullptr) {
    set_error("decode_layer_tail: null descriptor");
    return KVPR_EINVAL;
  }
  return layer_tail(*desc, static_cast<cudaStream_t>(stream));
}

int kvpr_decode_attention_kv4(const void* q, const void* kv_pages, const void* qpages, int q_lo, int q_hi, void* out,
                              void* ws, size_t ws_bytes, int batch, int heads, int head_dim, int seq_len, float scale,
                              void* stream) {
  g_err[0] = 0;
  return decode_attention_q4(static_cast<const __half*>(q), static_cast<const __half*>(kv_pages),
                             static_cast<const uint8_t*>(qpages), q_lo, q_hi, static_cast<__half*>(out),
                             static_cast<float*>(ws), ws_bytes, batch, heads, head_dim, seq_len, scale,
                             static_cast<cudaStream_t>(stream));
}

int kvpr_prefill_attention(const void* q, const void* kv_pages, void* out, int batch, int heads, int head_dim,
                           int seq_len, float scale, void* stream) {
  g_err[0] = 0;
  return prefill_attention(static_cast<const __half*>(q), static_cast<const __half*>(kv_pages),
                           static_cast<__half*>(out), batch, heads, head_dim, seq_len, scale,
                           static_cast<cudaStream_t>(stream));
}

int kvpr_layernorm(const float* x, long long ldx, const void* gamma, const void* beta, void* out, long long ldo,
                   int rows, int hidden, float eps, void* stream) {
  g_err[0] = 0;
  return layernorm(x, ldx, static_cast<const __half*>(gamma), static_cast<const __half*>(beta),
                   static_cast<__half*>(out), ldo, rows, hidden, eps, static_cast<cudaStream_t>(stream));
}

int kvpr_embed(const int* tokens, const void* tok_emb, const void* pos_emb, float* out, int rows, int batch,
               int pos_begin, int hidden, int pos_offset, void* stream) {
  g_err[0] = 0;
  return embed(tokens, static_cast<const __half*>(tok_emb), static_cast<const __half*>(pos_emb), out, rows, batch,
               pos_begin, hidden, pos_offset, static_cast<cudaStream_t>(stream));
}

int kvpr_argmax(const float* logits, long long ld, int rows, int cols, int* out_idx, float* out_val, void* stream) {
  g_err[0] = 0;
  return argmax_rows(logits, ld, rows, cols, out_idx, out_val, static_cast<cudaStream_t>(stream));
}

int kvpr_copy_batch_async(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t n, void* stream) {
  g_err[0] = 0;
  return copy_batch(dsts, srcs, sizes, n, static_cast<cudaStream_t>(stream));
}

int kvpr_copy_2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                       void* stream) {
  g_err[0] = 0;
  if (width == 0 || height == 0) return KVPR_OK;
  if (dst == nullptr || src == nullptr || dpitch < width || spitch < width) {
    set_error("copy_2d_async: null pointer or pitch < width");
    return KVPR_EINVAL;
  }
  cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("copy_2d_async: %s", cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}

int kvpr_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  g_err[0] = 0;
  if (bytes == 0) return KVPR_OK;
  if (dst == nullptr || src == nullptr) {
    set_error("copy_async: null pointer");
    return KVPR_EINVAL;
  }
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("copy_async: %s", cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}

size_t kvpr_kv4_page_bytes(int batch, int hidden) { return kv4_page_bytes(batch, hidden); }

int kvpr_kv4_quantize(const void* pages, void* qpages, int batch, int hidden, int pos_begin, int pos_end,
                      void* stream) {
  g_err[0] = 0;
  return kv4_quantize(static_cast<const __half*>(pages), static_cast<uint8_t*>(qpages), batch, hidden, pos_begin,
                      pos_end, static_cast<cudaStream_t>(stream));
}

int kvpr_kv4_dequantize(const void* qpages, void* pages, int batch, int hidden, int pos_begin, int pos_end,
                        void* stream) {
  g_err[0] = 0;
  return kv4_dequantize(static_cast<const uint8_t*>(qpages), static_cast<__half*>(pages), batch, hidden, pos_begin,
                        pos_end, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
