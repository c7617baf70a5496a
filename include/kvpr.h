/*
 * kvpr.h — C-ABI of libkvpr.so, the B200 (sm_100a) kernels behind KVPR's
 * per-layer decode path.
 *
 * The reference (`kvoverlap`, /root/reference/pkg) is a pure-Python planner
 * with no FFI; its numeric contract lives in numerics.py and its cost model
 * in costmodel.py / scheduler.py.  Each entry point below names the reference
 * routine whose semantics it takes over on the GPU.  The Python package
 * `paper_2411_17089_b200` binds these with ctypes (see _lib.py and
 * INTEGRATION.md) — that is the boundary a `kvoverlap` maintainer would bind.
 *
 * Conventions
 *  - The caller (Python / torch) owns every data buffer, device and pinned
 *    host.  The kernel entry points (K1-K8, the codec, the probes) borrow raw
 *    pointers: they never allocate or free memory and never synchronise; each
 *    launches on the caller's stream (`stream` is a cudaStream_t, NULL =
 *    legacy default stream) and returns once the launch is enqueued.
 *    The exceptions, all outside the per-step path and named here:
 *      * kvpr_decoder_create allocates the handle (host) and its CUDA events;
 *        kvpr_decoder_destroy frees them.  kvpr_decoder_run only enqueues.
 *      * kvpr_decoder_kernel_stats / kvpr_decoder_timeline wait on the
 *        timing events they read (cudaEventSynchronize), after a timed run.
 *      * kvpr_ipc_alloc / kvpr_ipc_free own the CUDA IPC peer regions of the
 *        TP all-reduce (cudaMalloc / cudaFree; IPC handles cannot wrap torch
 *        allocations); kvpr_ipc_open / _close map and unmap peers' regions.
 *      * the stream-K decode GEMM (kvpr_linear_ws, M <= 64) keeps per-tile
 *        arrival counters in a 16 KB zeroed device block the library
 *        allocates once per (device, stream) on first use; every call leaves
 *        them zero.  Workspaces (`ws`) are caller scratch of arbitrary
 *        contents; calls sharing a ws must be stream-ordered.
 *  - Return 0 on success.  KVPR_EINVAL (bad shape / pointer / range) maps to
 *    ValueError, as the reference raises ValueError for the same conditions
 *    (numerics.py:22-32, costmodel.py:31-43); KVPR_ECUDA maps to RuntimeError.
 *    kvpr_last_error() returns a thread-local message for the last failure.
 *  - fp16 storage, fp32 accumulation.  No CPU fallback exists: every entry
 *    point launches sm_100a code or fails.
 *
 * Layouts
 *  - KV pages (one layer): position-major slabs, page p = [2][batch][hidden]
 *    fp16 (K then V), i.e. element (p, kv, b, c) at ((p*2 + kv)*batch + b)*hidden + c.
 *    A contiguous position range [l, s) is therefore one contiguous byte
 *    range, so KV[l:s'-1] streams host->device as a single DMA.
 *  - Layer inputs X (post-LN1 activations, the recompute source): [pos][batch][hidden] fp16.
 *  - Linear weights: PyTorch layout [out_features, in_features] fp16 (K-major).
 */
#ifndef KVPR_H_
#define KVPR_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVPR_OK 0
#define KVPR_EINVAL 1
#define KVPR_ECUDA 2
#define KVPR_ECYCLE 3 /* kvpr_list_schedule: the dependency graph has a cycle */

/* epilogue flags for kvpr_linear */
#define KVPR_EPI_RELU 1  /* max(0, .) after bias */
#define KVPR_EPI_F32 2   /* fp32 output (default fp16) */
#define KVPR_EPI_ACCUM 4 /* fp32 output accumulated in place: out += result (residual add) */
#define KVPR_EPI_W_TILED 8 /* w is in kvpr_tile_weight's box-tiled layout (ldw ignored); decode GEMM, M <= 64 */

/* One output column segment of kvpr_linear.  Output element (m, n) with
 * seg = n / seg_width lands at
 *   ptr + (m % row_group) * ld + (m / row_group) * group_stride + n % seg_width
 * (elements of the output type). */
typedef struct kvpr_out_seg {
  void* ptr;
  long long group_stride;
} kvpr_out_seg;

typedef struct kvpr_epilogue {
  const void* bias;   /* fp16 [N] or NULL */
  int seg_width;      /* columns per segment, multiple of 32 */
  int row_group;      /* rows per group (>=1) */
  long long ld;       /* row stride inside a group, elements */
  kvpr_out_seg seg[3];
  float scale;        /* applied to columns [0, scale_cols) after the bias */
  int scale_cols;
  int flags;          /* KVPR_EPI_* */
} kvpr_epilogue;

/* Thread-local description of the last failure ("" if none). */
const char* kvpr_last_error(void);
/* Kernels this library has launched in this process (all entry points; for launch accounting). */
long long kvpr_kernel_launches(void);

/* ABI version (bumped on any signature change). */
int kvpr_version(void);

/* Number of SMs of `device` (for grid sizing in the host runtime). */
int kvpr_sm_count(int device);

/* K1 — recompute GEMM (tcgen05 + TMEM, TMA-fed).
 * Replaces numerics.split_merge_kv's prefix rebuild `X[:l] @ W_K`, `X[:l] @ W_V`
 * (numerics.py:129-133), with OPT's k_proj/v_proj biases, FLOPs per
 * costmodel.recompute_flops (costmodel.py:169-176).
 * For positions [pos_begin, pos_end):
 *   K[p, b, :] = X[p, b, :] . W_k^T + b_k,  V[p, b, :] = X[p, b, :] . W_v^T + b_v
 * written in place into the KV pages.
 *   x        : layer-input buffer, [pos][batch][hidden] fp16 (position 0 at x)
 *   w_kv     : [2*hidden, hidden] fp16 = rows of W_k then W_v (torch layout)
 *   b_kv     : [2*hidden] fp16 = b_k then b_v (may be NULL)
 *   kv_pages : page buffer of the layer, position 0 at kv_pages
 * pos_begin == pos_end is a no-op (split 0, numerics.py:127-128). */
int kvpr_recompute_kv(const void* x, const void* w_kv, const void* b_kv, void* kv_pages, int batch,
                      int pos_begin, int pos_end, int hidden, void* stream);

/* The tile kvpr_recompute_kv uses for a launch over `positions` positions on a GPU with `sms` SMs:
 * 512 = 256 x 256 CTA-pair tile (cta_group::2), 32..256 = 128 x BN tile on one CTA, 0 = invalid
 * arguments.  Pure host function (no CUDA call); the bench labels its roofline line with it. */
int kvpr_recompute_tile(int batch, int positions, int hidden, int sms);

/* Decode-weight layout: W [N, K] (row stride ldw) rewritten as [N/128][K/64][128][64] fp16, zero-padded
 * to whole 128 x 64 boxes, so each box the decode GEMM streams is 16 KB contiguous in HBM and a CTA's
 * k-range is one contiguous region (row-major boxes are 128 separate 128-byte runs, 8 KB apart).
 * Same products, same MMA order, same bits as the row-major operand.  out: kvpr_tiled_weight_bytes. */
size_t kvpr_tiled_weight_bytes(int N, int K);
int kvpr_tile_weight(const void* w, long long ldw, int N, int K, void* out, void* stream);

/* Fused projection: out = epilogue(A[M,K] . W[N,K]^T + bias), tcgen05 GEMM.
 * Used for the decode-token q/k/v (K3), out-proj + residual (K4), fc1+ReLU and
 * fc2 + residual (K6), LM head (K8), and the prefill that fills the host stores.
 * bn selects the tile: 32 / 64 / 128 / 256 = 128 x bn tile on one CTA; 512 = 256 x 256 tile on a
 * CTA pair (tcgen05 cta_group::2); -1 = weight-streaming decode GEMM with the operands swapped
 * (128 weight rows x all M <= 64 activation rows per tile); 0 = auto (-1 for M <= 64).  All
 * variants accumulate K in the same order, so without a K split they produce identical bits.
 * -2 = CUDA-core decode projection for M <= 8 (see kvpr_linear_ws; different k order). */
int kvpr_linear(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                const kvpr_epilogue* epi, int bn, void* stream);

/* kvpr_linear with an fp32 scratch buffer: single-row-block (decode) GEMMs may then split K
 * across CTAs (deterministic: partials reduced in slice order, then the same epilogue).
 * bn = -2 (and bn = 0 for M <= 8, unless KVPR_GEMV=0) selects the CUDA-core decode projection
 * (weight streaming with 16-byte loads, fixed reduction order): deterministic, but its k order
 * is not the tensor-core kernels', so the runtime never routes the q/k/v projection here. */
int kvpr_linear_ws(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                   const kvpr_epilogue* epi, int bn, void* ws, size_t ws_bytes, void* stream);

/* K5 + K6: y = LayerNorm(x) (fp32 rows [M][ldx] -> fp16 [M][ldy], as kvpr_layernorm) and
 * out = epilogue(y . W^T + bias) (as kvpr_linear_ws).  With KVPR_LN_FUSE=1 in the environment and
 * the projection on the CUDA-core path (bn -2, or auto at M <= 8) this is ONE launch: every CTA
 * normalises the rows into its staging buffer with kvpr_layernorm's exact arithmetic and CTA 0
 * stores y (measured slower than two launches at config 1, so not the default).  Otherwise the two
 * launches.  y and out are bit-identical to kvpr_layernorm followed by kvpr_linear_ws either way. */
int kvpr_layernorm_linear_ws(const float* x, long long ldx, const void* gamma, const void* beta, float eps, void* y,
                             long long ldy, const void* w, long long ldw, int M, int N, int K,
                             const kvpr_epilogue* epi, int bn, void* ws, size_t ws_bytes, void* stream);

/* K2 — split-KV decode attention over the merged cache, read in place.
 * Replaces numerics.decode_attention's per-head loop (numerics.py:166-190):
 * per (sequence b, head) softmax(scale * K q) V over positions [0, seq_len)
 * of the page buffer, max-subtracted softmax (numerics.py:159-163).  Positions
 * [0,l) hold recomputed K/V, [l, seq_len-1) the transferred tail, seq_len-1
 * the new token — one buffer, no concatenation.
 *   q   : [batch][hidden] fp16,  out : [batch][hidden] fp16 (heads concatenated)
 *   ws  : fp32 scratch for split partials; ws_bytes sizes the split count.
 * seq_len == 0 -> KVPR_EINVAL ("cannot attend over an empty cache"). */
int kvpr_decode_attention(const void* q, const void* kv_pages, void* out, void* ws, size_t ws_bytes, int batch,
                          int heads, int head_dim, int seq_len, float scale, void* stream);

/* K2 over a ragged batch: the reference keeps one KVState per sequence with its own length
 * (numerics.py:43-72).  Sequence b attends over positions [0, seq_lens[b]) of the same page
 * layout, padded to max_seq_len positions; seq_lens is a DEVICE int32[batch] with every entry in
 * [1, max_seq_len] (positions past a sequence's end are never read).  Same arithmetic as
 * kvpr_decode_attention when every length equals max_seq_len. */
int kvpr_decode_attention_ragged(const void* q, const void* kv_pages, const int* seq_lens, void* out, void* ws,
                                 size_t ws_bytes, int batch, int heads, int head_dim, int max_seq_len, float scale,
                                 void* stream);

/* K2 + K4 + K5 + K6 fused for small batches: the decode layer after its q/k/v projection, in ONE
 * cooperative kernel (one CTA per SM, grid-wide barriers between the stages):
 *   attn = decode_attention(q, pages[0, seq_len))            (as kvpr_decode_attention)
 *   hres += attn . W_o^T + b_o
 *   mid   = relu(LayerNorm2(hres) . W_1^T + b_1)
 *   hres += mid . W_2^T + b_2
 *   lnx_out = LayerNorm_x(hres)   (optional: the next layer's LN1 into its X slot, or the final LN)
 *   q_next, page_next = lnx_out . W_qkv_next^T + b_qkv_next   (optional: the next layer's K3)
 * The reference's decode_attention (numerics.py:166-191) followed by OPT's MLP block (SURVEY.md
 * §8a note 2).  Deterministic; agrees with the multi-kernel sequence to fp32 rounding (different
 * summation order).  Needs kvpr_decode_layer_tail_supported(); ws holds the attention split
 * partials (>= batch * heads * (head_dim + 2) * 4 bytes).  Grid-barrier words are a library-owned
 * zeroed block per (device, stream), made on first use; launches sharing a stream are ordered. */
typedef struct kvpr_layer_tail_desc {
  int batch, hidden, heads, head_dim, ffn, seq_len;
  float scale, eps;
  const void* q;        /* [batch][hidden] fp16 */
  const void* kv_pages; /* page buffer of the layer, positions [0, seq_len) */
  void* attn;           /* [batch][hidden] fp16 scratch (attention output) */
  const void *wo, *bo;
  float* hres;          /* [batch][hidden] fp32 residual stream, updated in place */
  const void *ln2_g, *ln2_b, *w1, *b1;
  void* mid;            /* [batch][ffn] fp16 scratch */
  const void *w2, *b2;
  const void *lnx_g, *lnx_b; /* optional output LayerNorm (NULL lnx_out = none) */
  void* lnx_out;
  long long lnx_ld;
  /* optional, with the output LayerNorm: the next layer's q/k/v of the new token from lnx_out
   * (K3 fused in): q -> q_next [batch][hidden], k, v -> page_next (K rows then V rows).  Same
   * k order as the tcgen05 kernels, so k, v are bit-identical to kvpr_linear / K1 (the split
   * invariance of numerics.split_merge_kv, numerics.py:107-137). */
  const void *wqkv_next, *bqkv_next; /* [3*hidden][hidden], [3*hidden] */
  void* q_next;
  void* page_next;
  /* optional zero-copy PCIe traffic (page-locked host stores, mapped): attention positions
   * [host_lo, host_hi) are read from kv_host (the layer's host KV store, same page layout) instead of
   * kv_pages -- the transferred tail KV[l:s'-1] without a copy-engine DMA; x_store_next /
   * page_store_next receive the normalised rows / the next layer's k, v page as well (the D2H
   * store_activation / store_cache of graph.py:340-347, written by the SMs). */
  const void* kv_host;
  int host_lo, host_hi;
  void* x_store_next;
  void* page_store_next;
  void* ws;
  size_t ws_bytes;
} kvpr_layer_tail_desc;

int kvpr_decode_layer_tail_supported(int batch, int hidden, int heads, int ffn);
int kvpr_decode_layer_tail(const kvpr_layer_tail_desc* desc, void* stream);

/* Causal attention for the prompt (prefill that populates the host stores):
 * q/out [pos][batch][hidden], kv pages as above, positions [0, seq_len).  head_dim 64 or 128,
 * batch * heads <= 65535 (else KVPR_EINVAL); one persistent launch of at most #SMs CTAs. */
int kvpr_prefill_attention(const void* q, const void* kv_pages, void* out, int batch, int heads, int head_dim,
                           int seq_len, float scale, void* stream);

/* K5 — LayerNorm of fp32 rows into fp16 (out row stride ldo). */
int kvpr_layernorm(const float* x, long long ldx, const void* gamma, const void* beta, void* out, long long ldo,
                   int rows, int hidden, float eps, void* stream);

/* K7 — token + learned position embedding into the fp32 residual stream.
 * Row r is (position pos_begin + r / batch, sequence r % batch). */
int kvpr_embed(const int* tokens, const void* tok_emb, const void* pos_emb, float* out, int rows, int batch,
               int pos_begin, int hidden, int pos_offset, void* stream);

/* K8 tail — per-row argmax (greedy token) of fp32 logits. */
int kvpr_argmax(const float* logits, long long ld, int rows, int cols, int* out_idx, float* out_val, void* stream);

/* Enqueue one DMA (cudaMemcpyAsync, direction inferred from UVA) on `stream`.
 * The runtime's H2D of X[:, :l] / KV[l:s'-1] and D2H of the new X row / K,V page
 * (pipesim graph.py:266-347 load_activation_recompute / load_cache /
 * store_activation / store_cache) go through here.  Host buffers must be
 * page-locked for the copy to be asynchronous. */
int kvpr_copy_async(void* dst, const void* src, size_t bytes, void* stream);

/* One strided DMA (cudaMemcpy2DAsync): `height` rows of `width` bytes, row r from src + r*spitch to
 * dst + r*dpitch.  The same prefix of several layers' stores (X[j][0:l] for consecutive layers j:
 * host pitch = one layer's store, device pitch = one staging buffer) in ONE copy-engine submission. */
int kvpr_copy_2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                       void* stream);

/* n (<= 16) DMAs enqueued in order on `stream`, one cudaMemcpyAsync each (zero-byte entries
 * skipped): the per-layer copies of a small model (X[:, :l] + KV[l:s'-1]; the new X row + K,V page)
 * in one C call. */
int kvpr_copy_batch_async(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t n, void* stream);

/* 4-bit groupwise KV pages (compressed KV offload; costmodel.py:109-118:
 * kv_bytes_per_element = 4/8 + 4/64 = 0.5625).  Compressed page = codes
 * [2][batch][hidden/2] bytes (element 2i low nibble) then params
 * [2][batch][hidden/64] x (fp16 min, fp16 scale); hidden % 64 == 0.
 * x^ = half(min + q*scale), q = clamp(rint((x - min)/scale), 0, 15). */
size_t kvpr_kv4_page_bytes(int batch, int hidden);

/* fp16 pages [pos_begin, pos_end) -> compressed pages (both buffers indexed from position 0). */
int kvpr_kv4_quantize(const void* pages, void* qpages, int batch, int hidden, int pos_begin, int pos_end,
                      void* stream);

/* compressed pages [pos_begin, pos_end) -> fp16 pages, in place for K2 to read. */
int kvpr_kv4_dequantize(const void* qpages, void* pages, int batch, int hidden, int pos_begin, int pos_end,
                        void* stream);

/* K2 over a mixed cache ("dequant fused into the staging read in K2"):
 * as kvpr_decode_attention, but positions [q_lo, q_hi) are read from 4-bit compressed pages
 * `qpages` (layout above, indexed from position 0) and dequantised in registers with the exact
 * arithmetic of kvpr_kv4_dequantize — identical bits to dequantize-then-K2, without writing the
 * fp16 tail to HBM and reading it back.  Other positions come from the fp16 pages. */
int kvpr_decode_attention_kv4(const void* q, const void* kv_pages, const void* qpages, int q_lo, int q_hi, void* out,
                              void* ws, size_t ws_bytes, int batch, int heads, int head_dim, int seq_len, float scale,
                              void* stream);

/* ---------------------------------------------------------------------------
 * Native decode executor: the per-layer issue loop of the Python runtime
 * (paper_2411_17089_b200/runtime.py, realising pipesim graph.py:232-347) in C,
 * one call per decode run.  Same kernels, launch parameters and event DAG as the
 * Python loop, hence identical results.  The caller owns every buffer; the handle
 * holds descriptors and CUDA events only. */
typedef struct kvpr_layer_desc {
  const void *ln1_g, *ln1_b, *wqkv, *bqkv, *wo, *bo, *ln2_g, *ln2_b, *w1, *b1, *w2, *b2;
  void* host_x;  /* pinned [capacity][batch][hidden] fp16 (unused when x_resident) */
  void* host_kv; /* pinned [capacity][2][batch][hidden] fp16 */
  void* dev_x;   /* x_resident: device [capacity][batch][hidden]; else NULL */
} kvpr_layer_desc;

typedef struct kvpr_decoder_desc {
  int layers, batch, hidden, heads, ffn, vocab, capacity, chunks, nbuf, x_resident;
  float eps;
  const void *embed, *pos, *lnf_g, *lnf_b;
  void* kv_dev; /* [nbuf][capacity][2][batch][hidden] fp16 */
  void* x_dev;  /* [nbuf][capacity][batch][hidden] fp16 */
  float* hres;  /* [batch][hidden] fp32 residual stream */
  void *q, *attn, *y, *mid, *zf;
  float* logits;
  int* tok;     /* [batch] int32: input tokens of the first step, then each step's greedy output */
  void* ws;
  size_t ws_bytes;
  void *compute_stream, *h2d_stream, *d2h_stream;
  int chunk_rows; /* minimum positions per X chunk / K1 launch (runtime.KVPRRuntime.chunk_rows) */
  int chunk_wave; /* > 0: X chunks are multiples of this many positions (whole K1 tile waves) */
  void* recompute_stream; /* non-NULL: K1 runs here, issued a unit ahead (overlaps the previous layer) */
  int fused_tail; /* 1: the layer after q/k/v is kvpr_decode_layer_tail (batch <= 8), LN1 / final LN fused into it */
  int zero_copy;  /* with fused_tail: bit 0 = the tail reads KV[l:s'-1] from the host store (no KV DMA),
                     bit 1 = it writes the next unit's X row / k,v page to the host stores (no D2H DMAs) */
  int dma_group;  /* > 1: the KV-tail copies KV[l:s'-1] of dma_group consecutive layers of a step (single
                     X chunk or X resident) go as ONE strided 2-D DMA -- the copy engine's ~4 us fixed
                     cost per submission is paid once per group (X stays one DMA per layer, so each
                     K1 waits only for its own rows).  Needs layers % dma_group == 0, layers >=
                     2 * dma_group, nbuf >= 2 * dma_group, nbuf % dma_group == 0 and equally spaced
                     per-layer host KV stores; otherwise (or <= 1) one KV DMA per layer. */
} kvpr_decoder_desc;

int kvpr_decoder_create(const kvpr_decoder_desc* desc, const kvpr_layer_desc* layers, void** handle);
int kvpr_decoder_destroy(void* handle);
/* steps decode steps from cache length base_len with per-step splits; tokens of step i land in
 * out_tokens[i][batch] (device, may be NULL), logits in out_logits[i][batch][vocab] (may be NULL). */
int kvpr_decoder_run(void* handle, int base_len, const int* splits, int steps, int* out_tokens, float* out_logits);

/* Bracket every K1 (kind 0) / K2 (kind 1) launch of subsequent runs with CUDA timing events
 * (enable=0 clears them); stats: launches, mean seconds per launch, mean algorithmic units
 * (FLOPs for K1, bytes for K2) per launch.  Synchronises on the recorded events. */
int kvpr_decoder_set_timing(void* handle, int enable);
int kvpr_decoder_kernel_stats(void* handle, int kind, int* launches, double* mean_seconds, double* mean_units);
/* Timeline of the last timed run, in runtime.DecodeTiming's convention: layer_ms[i*layers+j] =
 * compute-stream time from the previous layer end (or step i's start) to the end of layer j of
 * step i; step_ms[i] = time from the previous step's end (or the run start) to the end of step
 * i's head.  Returns the number of steps (0 if the last run was untimed), or -KVPR_E* on error. */
int kvpr_decoder_timeline(void* handle, float* layer_ms, int layer_cap, float* step_ms, int step_cap);
/* Kernel launches (ABI-level) the executor has issued so far. */
long long kvpr_decoder_launches(void* handle);

/* Compiled engine of the pipeline simulator (kvoverlap.pipesim's _engine.pyx, engine.py:45-76): list
 * scheduling of n tasks onto n_resources exclusive lanes, dependencies as CSR (task i waits for
 * dep_indices[dep_indptr[i] .. dep_indptr[i+1])); fills start / end.  Host code, no GPU.  Returns
 * KVPR_ECYCLE when some tasks never become ready. */
int kvpr_list_schedule(long long n, const long long* resource, const double* duration, const long long* priority,
                       const long long* dep_indptr, const long long* dep_indices, int n_resources, double* start,
                       double* end);

/* ---------------------------------------------------------------------------------------------
 * Fused tensor-parallel projection + all-reduce over peer memory (config 4: head-sharded OPT-30B;
 * replaces the reference-less NCCL all-reduce after the row-parallel out-proj / fc2).
 * Peer buffers are CUDA IPC allocations: every rank allocates one region with kvpr_ipc_alloc,
 * the host exchanges the handles (torch.distributed object all-gather) and opens the peers'
 * regions with kvpr_ipc_open (cudaIpcMemLazyEnablePeerAccess: NVLink P2P between GPUs). */
/* Diagnostic only (tools/k2_probe.py): host -> device copy by SM loads from page-locked host memory. */
int kvpr_debug_sm_pull(const void* host, void* dev, size_t bytes, int ctas, void* stream);

#define KVPR_TP_MAX_WORLD 8
#define KVPR_TP_MAX_TILES 512

typedef struct kvpr_tp_peers {
  int rank, world;                     /* 2 <= world <= KVPR_TP_MAX_WORLD */
  void* recv[KVPR_TP_MAX_WORLD];       /* every rank's receive slots: [world][M][N] fp32 */
  float* resid[KVPR_TP_MAX_WORLD];     /* every rank's residual [M][N] fp32 (identical before the call) */
  unsigned* flags[KVPR_TP_MAX_WORLD];  /* every rank's flags: [world][512] push + [512] broadcast, zeroed once */
  unsigned* err;                       /* this rank's error word: nonzero after a peer wait timed out (5 s) */
} kvpr_tp_peers;

size_t kvpr_ipc_handle_bytes(void);
/* cudaMalloc + zero + cudaIpcGetMemHandle; handle receives kvpr_ipc_handle_bytes() bytes */
int kvpr_ipc_alloc(size_t bytes, void** dptr, void* handle);
int kvpr_ipc_open(const void* handle, void** dptr);
int kvpr_ipc_close(void* dptr);
int kvpr_ipc_free(void* dptr);

/* On every rank r of peers->world, with the same residual R on all ranks before the call:
 *   R[m, n] <- R[m, n] + (sum_r A_r[m, :] . W_r[n, :] + bias[n])     (M <= 64, fp32 residual)
 * A_r [M, K] fp16 and W_r [N, K] fp16 are rank r's K slices (row-parallel weights).  Two kernels on
 * `stream`: the swap-AB GEMM pushing each 128-column tile's partial to its owner (tile % world), and
 * the owners' rank-ordered sum + broadcast into every residual (deterministic).  `epoch` must grow
 * by one per call on every rank (same value on all ranks).  Replaces kvpr_linear_ws + all-reduce. */
int kvpr_linear_allreduce(const void* a, long long lda, const void* w, long long ldw, int M, int N, int K,
                          const void* bias, const kvpr_tp_peers* peers, unsigned epoch, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KVPR_H_ */
