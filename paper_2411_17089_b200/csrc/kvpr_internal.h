// Internal (C++) declarations shared between the kernel translation units and
// the extern "C" boundary in abi.cu.  Nothing here crosses the C-ABI.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kvpr.h"

namespace kvpr {

constexpr int kTpMaxWorld = 8;     // ranks of one fused TP all-reduce (one NVSwitch domain slice)
constexpr int kTpMaxTiles = 512;   // 128-column tiles of N per fused all-reduce (N <= 65536)

// Epilogue + shape bundle for the tcgen05 GEMM (passed by value as a kernel arg).
//   out address of (m, n) = seg_ptr[n / seg_width]
//                         + (m % row_group) * ld + (m / row_group) * seg_group_stride[seg]
//                         + (n % seg_width)
struct GemmArgs {
  int M, N, K;
  int num_m_blk, num_n_blk, num_k_blk;
  const __half* bias;
  int seg_width;
  int row_group;
  long long ld;
  void* seg_ptr[3];
  long long seg_group_stride[3];
  float scale;
  int scale_cols;
  int flags;
  int a_box_rows;  // rows of A per TMA box (128, or M rounded up to 8 for single-tile small-M GEMMs)
  int k_splits;    // > 1: each CTA reduces a K slice into ws; a second kernel applies the epilogue
  float* ws;       // split-K partials [k_splits][M][ws_ld] fp32
  int ws_ld;
  int group_m;     // rasterization band (tile_coords): > 0 m-blocks per band, < 0 n-blocks per band
  // stream-K swap-AB decode GEMM (sk_ctas > 0): CTAs; fp32 partial slots in ws; per-tile arrival
  // counters (library-owned, zero between calls)
  int sk_ctas;
  unsigned* sk_counters;
  int w_tiled;  // swap-AB: W in the box-tiled layout of kvpr_tile_weight (each 128 x 64 box contiguous)
  int max_ctas;  // > 0: persistent tcgen05 GEMMs use at most this many CTAs (SMs left to a concurrent kernel)
  // fused TP all-reduce (swap-AB kernel only; tp_world > 1): raw partials pushed to the tile owner
  int tp_rank, tp_world;
  unsigned tp_epoch;
  float* tp_recv[kTpMaxWorld];     // per rank: receive slots [world][M][N] fp32
  unsigned* tp_flags[kTpMaxWorld];  // per rank: push flags [world][kTpMaxTiles]
};

int sm_count(int device);
void clear_error();
int copy_batch(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t n, cudaStream_t stream);



// CUDA-core projection for decode batches M <= kGemvMaxM (gemv.cu); deterministic, but not the
// tensor-core kernels' k order (never used for outputs K1 rebuilds)
constexpr int kGemvMaxM = 8;
constexpr int kGemvMaxSmem = 96 * 1024;  // activations staged per CTA: M * K * 2 bytes
constexpr int kGemvLnMaxK = 2048;        // LN prologue holds a row in 2 float4 per thread
size_t gemv_smem_bytes(int M, int K);
struct GemvLn {  // LayerNorm prologue of the fused decode projection (A = LN(x) rows)
  const float* x;
  long long ldx;
  const __half* gamma;
  const __half* beta;
  float eps;
  __half* y;  // LN output [M][ldy], written by CTA 0 (may be null)
  long long ldy;
};
int gemv_f16(const void* a, long long lda, const void* w, long long ldw, const GemmArgs& args, cudaStream_t stream,
             const GemvLn* ln = nullptr);
int gemv_slices(int N, int device);

// rank-2..5 fp16 tensor map with the 128-byte swizzle (gemm_tcgen05.cu); strides in bytes for dims 1..
int make_tmap_nd(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                 const uint32_t* box);

int gemm_f16(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K, const GemmArgs& epi,
             int bn, cudaStream_t stream, float* ws = nullptr, size_t ws_bytes = 0, const GemvLn* ln = nullptr);

size_t tiled_weight_bytes(int N, int K);
int tile_weight(const void* w, long long ldw, int N, int K, void* out, cudaStream_t stream);

int gemm_tp_partials(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                     const GemmArgs& tp, cudaStream_t stream);

// seq_lens (device int32[batch], optional): ragged batch, sequence b attends over [0, seq_lens[b])
int decode_attention(const __half* q, const __half* kv, __half* out, float* ws, size_t ws_bytes, int batch,
                     int heads, int head_dim, int seq_len, float scale, cudaStream_t stream,
                     const int* seq_lens = nullptr);

int decode_attention_q4(const __half* q, const __half* kv, const uint8_t* qpages, int q_lo, int q_hi, __half* out,
                        float* ws, size_t ws_bytes, int batch, int heads, int head_dim, int seq_len, float scale,
                        cudaStream_t stream, const int* seq_lens = nullptr);

bool layer_tail_supported(int batch, int hidden, int heads, int ffn);
int layer_tail(const kvpr_layer_tail_desc& d, cudaStream_t stream);

int prefill_attention(const __half* q, const __half* kv, __half* out, int batch, int heads, int head_dim,
                      int seq_len, float scale, cudaStream_t stream);

int layernorm(const float* x, long long ldx, const __half* gamma, const __half* beta, __half* out, long long ldo,
              int rows, int hidden, float eps, cudaStream_t stream);

int embed(const int* tokens, const __half* tok_emb, const __half* pos_emb, float* out, int rows, int batch,
          int pos_begin, int hidden, int pos_offset, cudaStream_t stream);

int argmax_rows(const float* logits, long long ld, int rows, int cols, int* out_idx, float* out_val,
                cudaStream_t stream);

size_t kv4_page_bytes(int batch, int hidden);
int kv4_quantize(const __half* pages, uint8_t* qpages, int batch, int hidden, int pos_begin, int pos_end,
                 cudaStream_t stream);
int kv4_dequantize(const uint8_t* qpages, __half* pages, int batch, int hidden, int pos_begin, int pos_end,
                   cudaStream_t stream);

}  // namespace kvpr
