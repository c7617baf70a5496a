// Native decode executor: the per-layer issue loop of runtime.KVPRRuntime.decode in C++.
//
// Same DAG, same kernels, same launch parameters as the Python loop (so the two produce
// identical bits, tests/test_executor_gpu.py), but one C call per decode run instead of
// ~30 Python->C calls per layer — the loop costs ~microseconds per layer of host time, which
// is what lets small models (BASELINE config 1) run at PCIe speed rather than at Python speed.
//
// Per unit u = (step i, layer j), buffer u % nbuf (graph.py:215-221 double buffering):
//   H2D stream : [wait compute(u-nbuf), D2H(u-nbuf), D2H(u-L)] X chunks -> x_dev, KV tail -> kv_dev
//   compute    : LN1 -> q,k,v (k,v into page s'-1) -> K1 per landed chunk -> [KV] K2 -> out-proj
//                -> LN2 -> fc1 -> fc2 ; head on the last layer
//   D2H stream : new X row, new K,V page -> host stores
// The caller owns every buffer (the handle holds only descriptors and CUDA events).

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "kvpr_internal.h"

#define KV_TRY(x)        \
  do {                   \
    int _rc = (x);       \
    if (_rc) return _rc; \
  } while (0)

namespace kvpr {

namespace {

struct KTime {
  int kind;  // 0 = K1 recompute GEMM, 1 = K2 decode attention, 2 = one H2D DMA (units = bytes)
  double units;
  cudaEvent_t a, b;
};

struct Decoder {
  kvpr_decoder_desc d;
  std::vector<kvpr_layer_desc> layer;
  int R = 0;
  std::vector<cudaEvent_t> ev_x, ev_kv, ev_qkv, ev_d2h, ev_done, ev_k1;  // ring of R units (ev_x: R*chunks)
  bool timing = false;  // bracket K1 / K2 launches with timing events (kvpr_decoder_kernel_stats)
  std::vector<KTime> kt;
  std::vector<cudaEvent_t> pool;  // timing events, created once and reused across runs
  size_t pool_used = 0;
  cudaEvent_t t0 = nullptr;                          // run start (timing only)
  std::vector<cudaEvent_t> layer_marks, step_marks;  // after each layer / after each step's head

  long long launches = 0;
  int group = 1;                            // layers per KV-tail DMA (kvpr_decoder_desc.dma_group, validated)
  long long host_kv_pitch = 0;              // bytes between consecutive layers' host KV stores
};

inline int pool_take(Decoder& D, cudaEvent_t* e) {
  if (D.pool_used == D.pool.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t x;
      if (cudaEventCreate(&x) != cudaSuccess) {
        set_error("timing event create failed");
        return KVPR_ECUDA;
      }
      D.pool.push_back(x);
    }
  }
  *e = D.pool[D.pool_used++];
  return KVPR_OK;
}

inline int kt_begin(Decoder& D, int kind, double units, cudaStream_t s, KTime* out) {
  if (!D.timing) return KVPR_OK;
  out->kind = kind;
  out->units = units;
  KV_TRY(pool_take(D, &out->a));
  KV_TRY(pool_take(D, &out->b));
  return cudaEventRecord(out->a, s) == cudaSuccess ? KVPR_OK : KVPR_ECUDA;
}

inline int kt_end(Decoder& D, KTime* t, cudaStream_t s) {
  if (!D.timing) return KVPR_OK;
  if (cudaEventRecord(t->b, s) != cudaSuccess) return KVPR_ECUDA;
  D.kt.push_back(*t);
  return KVPR_OK;
}

// timing only: one event on the compute stream, appended to `marks`
inline int mark(Decoder& D, std::vector<cudaEvent_t>& marks, cudaStream_t s) {
  if (!D.timing) return KVPR_OK;
  cudaEvent_t e;
  KV_TRY(pool_take(D, &e));
  if (cudaEventRecord(e, s) != cudaSuccess) return KVPR_ECUDA;
  marks.push_back(e);
  return KVPR_OK;
}

inline int ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return KVPR_ECUDA;
  }
  return KVPR_OK;
}


// chunk_bounds() of runtime.py: <= chunks contiguous ranges of >= min_rows positions when possible;
// with wave > 0 (and n >= wave) every range but the last is a multiple of wave positions
inline int chunk_bounds(int n, int chunks, int (*out)[2], int min_rows = 64, int wave = 0) {
  if (n <= 0) return 0;
  if (wave > 0 && n >= wave) {
    const int waves = (n + wave - 1) / wave;
    int per = wave * ((waves + chunks - 1) / chunks);
    const int min_per = wave * ((min_rows + wave - 1) / wave);
    if (per < min_per) per = min_per;
    int c = 0;
    for (int p = 0; p < n; p += per, ++c) {
      out[c][0] = p;
      out[c][1] = p + per < n ? p + per : n;
    }
    if (c > 1 && out[c - 1][1] - out[c - 1][0] < per / 2) {  // a short tail rides on the last chunk
      out[c - 2][1] = n;
      --c;
    }
    return c;
  }
  int c = n >= min_rows ? n / min_rows : 1;
  if (c > chunks) c = chunks;
  if (c < 1) c = 1;
  const int base = n / c, rem = n % c;
  int p = 0;
  for (int i = 0; i < c; ++i) {
    const int q = p + base + (i < rem ? 1 : 0);
    out[i][0] = p;
    out[i][1] = q;
    p = q;
  }
  return c;
}

inline int chunk_rows(const kvpr_decoder_desc& d) { return d.chunk_rows > 0 ? d.chunk_rows : 64; }

kvpr_epilogue simple_epi(void* out, long long ld, int M, int N, const void* bias, int flags) {
  kvpr_epilogue e;
  memset(&e, 0, sizeof(e));
  e.bias = bias;
  e.seg_width = ((N + 31) / 32) * 32;
  e.row_group = M;
  e.ld = ld;
  e.seg[0].ptr = out;
  e.scale = 1.f;
  e.flags = flags;
  return e;
}

struct Unit {
  int i, j, s, lp, buf, r;
};

inline Unit unit_of(const Decoder& D, int u, int base, const int* splits) {
  const int L = D.d.layers;
  Unit x;
  x.i = u / L;
  x.j = u % L;
  x.s = base + x.i + 1;
  x.lp = splits[x.i] < x.s - 1 ? splits[x.i] : x.s - 1;
  x.buf = u % D.d.nbuf;
  x.r = u % D.R;
  return x;
}

// one H2D DMA on hs, bracketed by timing events in timed runs (kvpr_decoder_kernel_stats kind 2)
int h2d(Decoder& D, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
        cudaStream_t hs, const char* what) {
  KTime t;
  KV_TRY(kt_begin(D, 2, static_cast<double>(width) * height, hs, &t));
  if (height == 1)
    KV_TRY(ck(cudaMemcpyAsync(dst, src, width, cudaMemcpyDefault, hs), what));
  else
    KV_TRY(ck(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, hs), what));
  return kt_end(D, &t, hs);
}

int issue_h2d(Decoder& D, int u, int base, const int* splits) {
  const kvpr_decoder_desc& d = D.d;
  const Unit x = unit_of(D, u, base, splits);
  cudaStream_t hs = static_cast<cudaStream_t>(d.h2d_stream);
  if (u >= d.nbuf) {
    const int rp = (u - d.nbuf) % D.R;
    KV_TRY(ck(cudaStreamWaitEvent(hs, D.ev_done[rp], 0), "wait compute"));
    KV_TRY(ck(cudaStreamWaitEvent(hs, D.ev_d2h[rp], 0), "wait d2h"));
  }
  if (u >= d.layers) KV_TRY(ck(cudaStreamWaitEvent(hs, D.ev_d2h[(u - d.layers) % D.R], 0), "wait store"));
  const size_t row = static_cast<size_t>(d.batch) * d.hidden * 2;
  const kvpr_layer_desc& Lw = D.layer[x.j];
  char* xd = static_cast<char*>(d.x_dev) + static_cast<size_t>(x.buf) * d.capacity * row;
  char* kvd = static_cast<char*>(d.kv_dev) + static_cast<size_t>(x.buf) * d.capacity * 2 * row;
  const bool kv_dma = x.s - 1 > x.lp && !(d.fused_tail && (d.zero_copy & 1));  // else the tail reads it itself
  void* kv_dst = kvd + x.lp * 2 * row;
  const void* kv_src = static_cast<const char*>(Lw.host_kv) + x.lp * 2 * row;
  const size_t kv_bytes = kv_dma ? (x.s - 1 - x.lp) * 2 * row : 0;
  int cb[16][2];
  const int nc = d.x_resident ? 0 : chunk_bounds(x.lp, d.chunks, cb, chunk_rows(d), d.chunk_wave);
  if (D.group > 1 && nc <= 1) {
    // small layers: X per unit (K1 of unit u waits only for its own rows), the KV tails of layers
    // [j, j + G) of this step (same s', l) as ONE strided DMA issued by the group's leader (j % G == 0)
    // after every member's buffer-reuse and store waits -- the members' staging buffers are
    // consecutive (nbuf % G == 0) and their host stores equally spaced.  A ~0.1 MB tail costs ~1.8 us
    // of PCIe and ~3.7 us of copy-engine overhead on its own (profiles/r02_dma_2d_probe.json)
    const int G = D.group;
    if (nc == 1) {
      KV_TRY(h2d(D, xd, 0, Lw.host_x, 0, static_cast<size_t>(cb[0][1] - cb[0][0]) * row, 1, hs, "h2d X"));
      KV_TRY(ck(cudaEventRecord(D.ev_x[x.r * d.chunks], hs), "record X"));
    }
    if (u % G != 0) return KVPR_OK;  // KV issued (and ev_kv recorded) by the leader
    for (int g = 1; g < G; ++g) {
      const int v = u + g;
      if (v >= d.nbuf) {
        const int rp = (v - d.nbuf) % D.R;
        KV_TRY(ck(cudaStreamWaitEvent(hs, D.ev_done[rp], 0), "wait compute"));
        KV_TRY(ck(cudaStreamWaitEvent(hs, D.ev_d2h[rp], 0), "wait d2h"));
      }
      if (v >= d.layers) KV_TRY(ck(cudaStreamWaitEvent(hs, D.ev_d2h[(v - d.layers) % D.R], 0), "wait store"));
    }
    if (kv_bytes)
      KV_TRY(h2d(D, kv_dst, 2 * static_cast<size_t>(d.capacity) * row, kv_src, static_cast<size_t>(D.host_kv_pitch),
                 kv_bytes, G, hs, "h2d KV (grouped)"));
    for (int g = 1; g < G; ++g) KV_TRY(ck(cudaEventRecord(D.ev_kv[(u + g) % D.R], hs), "record KV"));
    return ck(cudaEventRecord(D.ev_kv[x.r], hs), "record KV");
  }
  for (int c = 0; c < nc; ++c) {
    KV_TRY(h2d(D, xd + cb[c][0] * row, 0, static_cast<const char*>(Lw.host_x) + cb[c][0] * row, 0,
               (cb[c][1] - cb[c][0]) * row, 1, hs, "h2d X"));
    KV_TRY(ck(cudaEventRecord(D.ev_x[x.r * d.chunks + c], hs), "record X"));
  }
  if (kv_bytes) KV_TRY(h2d(D, kv_dst, 0, kv_src, 0, kv_bytes, 1, hs, "h2d KV"));
  return ck(cudaEventRecord(D.ev_kv[x.r], hs), "record KV");
}

// K1 chunks of unit x on stream st, each after its X chunk landed
int issue_k1_on(Decoder& D, const Unit& x, __half* xd, __half* kvd, cudaStream_t st) {
  const kvpr_decoder_desc& d = D.d;
  const kvpr_layer_desc& Lw = D.layer[x.j];
  const int b = d.batch, h = d.hidden;
  int cb[16][2];
  const int nc = chunk_bounds(x.lp, d.x_resident ? 1 : d.chunks, cb, chunk_rows(d), d.x_resident ? 0 : d.chunk_wave);
  const __half* wkv = static_cast<const __half*>(Lw.wqkv) + static_cast<size_t>(h) * h;
  const __half* bkv = static_cast<const __half*>(Lw.bqkv) + h;
  for (int c = 0; c < nc; ++c) {
    if (!d.x_resident) KV_TRY(ck(cudaStreamWaitEvent(st, D.ev_x[x.r * d.chunks + c], 0), "wait X chunk"));
    KTime t;
    KV_TRY(kt_begin(D, 0, 4.0 * b * (cb[c][1] - cb[c][0]) * static_cast<double>(h) * h, st, &t));
    KV_TRY(kvpr_recompute_kv(xd, wkv, bkv, kvd, b, cb[c][0], cb[c][1], h, st));
    KV_TRY(kt_end(D, &t, st));
  }
  return KVPR_OK;
}

// K1 of unit u on the recompute stream, issued one unit ahead of its layer's compute so the rebuild
// overlaps the previous layer's tail (small models: the layer chain is latency bound).  Hazards on
// buffer u % nbuf: its pages [0, l) were last read by K2(u - nbuf) (ev_done) and by the D2H of
// unit u - nbuf, which copies that unit's new page s_prev - 1 to the host store (ev_d2h).  When
// u - nbuf belongs to the previous step (layer j < nbuf), s_prev - 1 = s' - 2 lies inside [0, l)
// whenever l >= s' - 1, so K1 must not start before that copy has read the page.  The streamed-X
// H2D of u already waits on both, and so do its chunk events, but the X-resident path has no H2D
// and has to wait itself.  Its X rows come from the H2D of u or, X resident, from LN1 of the same
// layer one step back (ev_qkv).
int issue_k1(Decoder& D, int u, int base, const int* splits) {
  const kvpr_decoder_desc& d = D.d;
  const Unit x = unit_of(D, u, base, splits);
  cudaStream_t rs = static_cast<cudaStream_t>(d.recompute_stream);
  if (u >= d.nbuf) {
    KV_TRY(ck(cudaStreamWaitEvent(rs, D.ev_done[(u - d.nbuf) % D.R], 0), "k1 wait buffer"));
    KV_TRY(ck(cudaStreamWaitEvent(rs, D.ev_d2h[(u - d.nbuf) % D.R], 0), "k1 wait page store"));
  }
  if (d.x_resident && u >= d.layers)
    KV_TRY(ck(cudaStreamWaitEvent(rs, D.ev_qkv[(u - d.layers) % D.R], 0), "k1 wait X row"));
  const long long bh = static_cast<long long>(d.batch) * d.hidden;
  const kvpr_layer_desc& Lw = D.layer[x.j];
  __half* xd = d.x_resident ? static_cast<__half*>(Lw.dev_x)
                            : static_cast<__half*>(d.x_dev) + static_cast<size_t>(x.buf) * d.capacity * bh;
  __half* kvd = static_cast<__half*>(d.kv_dev) + static_cast<size_t>(x.buf) * d.capacity * 2 * bh;
  KV_TRY(issue_k1_on(D, x, xd, kvd, rs));
  return ck(cudaEventRecord(D.ev_k1[x.r], rs), "record K1");
}

int head(Decoder& D, cudaStream_t cs) {
  const kvpr_decoder_desc& d = D.d;
  if (!d.fused_tail)  // fused: the last layer's tail already wrote LN_f(h) into zf
    KV_TRY(layernorm(d.hres, d.hidden, static_cast<const __half*>(d.lnf_g), static_cast<const __half*>(d.lnf_b),
                     static_cast<__half*>(d.zf), d.hidden, d.batch, d.hidden, d.eps, cs));
  kvpr_epilogue e = simple_epi(d.logits, d.vocab, d.batch, d.vocab, nullptr, KVPR_EPI_F32);
  KV_TRY(kvpr_linear_ws(d.zf, d.hidden, d.embed, d.hidden, d.batch, d.vocab, d.hidden, &e, 0, d.ws, d.ws_bytes, cs));
  return argmax_rows(d.logits, d.vocab, d.batch, d.vocab, d.tok, nullptr, cs);
}

// Small batches: K2 -> out-proj -> LN2 -> fc1 -> fc2 as ONE cooperative kernel (layer_tail.cu), which
// also normalises the new residual into the next layer's X slot and computes that layer's q, k, v of
// the new token (K3, bit-identical to kvpr_linear) -- or, after the last layer, the final LN into zf.
// The next unit's X slot and page s'-1 were last read by the D2H of unit u + 1 - nbuf, so that copy
// must be done before this launch.
int fused_tail(Decoder& D, int u, const Unit& x, __half* kvd, cudaStream_t cs) {
  const kvpr_decoder_desc& d = D.d;
  const kvpr_layer_desc& Lw = D.layer[x.j];
  const int b = d.batch, h = d.hidden;
  const long long bh = static_cast<long long>(b) * h;
  kvpr_layer_tail_desc t;
  memset(&t, 0, sizeof(t));
  t.batch = b;
  t.hidden = h;
  t.heads = d.heads;
  t.head_dim = h / d.heads;
  t.ffn = d.ffn;
  t.seq_len = x.s;
  t.scale = static_cast<float>(1.0 / sqrt(static_cast<double>(h / d.heads)));
  t.eps = d.eps;
  t.q = d.q;
  t.kv_pages = kvd;
  t.attn = d.attn;
  t.wo = Lw.wo;
  t.bo = Lw.bo;
  t.hres = d.hres;
  t.ln2_g = Lw.ln2_g;
  t.ln2_b = Lw.ln2_b;
  t.w1 = Lw.w1;
  t.b1 = Lw.b1;
  t.mid = d.mid;
  t.w2 = Lw.w2;
  t.b2 = Lw.b2;
  t.lnx_ld = h;
  if (x.j + 1 < d.layers) {
    const kvpr_layer_desc& Ln = D.layer[x.j + 1];  // unit u + 1: same step, next layer, buffer (u + 1) % nbuf
    const size_t nb = static_cast<size_t>((u + 1) % d.nbuf);
    __half* xn = d.x_resident ? static_cast<__half*>(Ln.dev_x) : static_cast<__half*>(d.x_dev) + nb * d.capacity * bh;
    __half* kvn = static_cast<__half*>(d.kv_dev) + nb * d.capacity * 2 * bh;
    if (u + 1 >= d.nbuf) KV_TRY(ck(cudaStreamWaitEvent(cs, D.ev_d2h[(u + 1 - d.nbuf) % D.R], 0), "wait d2h (next slot)"));
    t.lnx_g = Ln.ln1_g;
    t.lnx_b = Ln.ln1_b;
    t.lnx_out = xn + static_cast<size_t>(x.s - 1) * bh;
    t.wqkv_next = Ln.wqkv;
    t.bqkv_next = Ln.bqkv;
    t.q_next = d.q;
    t.page_next = kvn + static_cast<size_t>(x.s - 1) * 2 * bh;
    if (d.zero_copy & 2) {
      t.x_store_next = d.x_resident ? nullptr : static_cast<__half*>(Ln.host_x) + static_cast<size_t>(x.s - 1) * bh;
      t.page_store_next = static_cast<__half*>(Ln.host_kv) + static_cast<size_t>(x.s - 1) * 2 * bh;
    }
  } else {
    t.lnx_g = d.lnf_g;
    t.lnx_b = d.lnf_b;
    t.lnx_out = d.zf;
  }
  // KV[l:s'-1] straight from the host store (zero-copy over PCIe); its last position was stored by
  // unit u - L (the previous step of this layer)
  if (x.s - 1 > x.lp && (d.zero_copy & 1)) {
    if (u >= d.layers) KV_TRY(ck(cudaStreamWaitEvent(cs, D.ev_d2h[(u - d.layers) % D.R], 0), "wait store (tail)"));
    t.kv_host = Lw.host_kv;
    t.host_lo = x.lp;
    t.host_hi = x.s - 1;
  }
  t.ws = d.ws;
  t.ws_bytes = d.ws_bytes;
  KTime t2;
  KV_TRY(kt_begin(D, 1, 2.0 * b * x.s * static_cast<double>(h) * 2, cs, &t2));
  KV_TRY(layer_tail(t, cs));
  KV_TRY(kt_end(D, &t2, cs));
  return ck(cudaEventRecord(D.ev_done[x.r], cs), "record done");
}

int compute(Decoder& D, int u, int base, const int* splits) {
  const kvpr_decoder_desc& d = D.d;
  const Unit x = unit_of(D, u, base, splits);
  const kvpr_layer_desc& Lw = D.layer[x.j];
  cudaStream_t cs = static_cast<cudaStream_t>(d.compute_stream);
  cudaStream_t ds = static_cast<cudaStream_t>(d.d2h_stream);
  const int b = d.batch, h = d.hidden;
  const long long bh = static_cast<long long>(b) * h;
  const size_t row = static_cast<size_t>(bh) * 2;
  __half* xd = d.x_resident ? static_cast<__half*>(Lw.dev_x)
                            : static_cast<__half*>(d.x_dev) + static_cast<size_t>(x.buf) * d.capacity * bh;
  __half* kvd = static_cast<__half*>(d.kv_dev) + static_cast<size_t>(x.buf) * d.capacity * 2 * bh;
  __half* x_slot = xd + static_cast<size_t>(x.s - 1) * bh;
  __half* page = kvd + static_cast<size_t>(x.s - 1) * 2 * bh;
  if (u >= d.nbuf) KV_TRY(ck(cudaStreamWaitEvent(cs, D.ev_d2h[(u - d.nbuf) % D.R], 0), "wait d2h (slot reuse)"));
  if (x.j == 0) {
    KV_TRY(embed(d.tok, static_cast<const __half*>(d.embed), static_cast<const __half*>(d.pos), d.hres, b, b,
                 x.s - 1, h, 2, cs));
  }
  // new token: LN1 into the X slot of position s'-1; q / k,v (k,v into page s'-1)
  const bool own_qkv = !d.fused_tail || x.j == 0;  // fused: the previous layer's tail made LN1 and q, k, v
  if (own_qkv)
    KV_TRY(layernorm(d.hres, h, static_cast<const __half*>(Lw.ln1_g), static_cast<const __half*>(Lw.ln1_b), x_slot, h,
                     b, h, d.eps, cs));
  if (own_qkv) {
    kvpr_epilogue e;
    memset(&e, 0, sizeof(e));
    e.bias = Lw.bqkv;
    e.seg_width = h;
    e.row_group = b;
    e.ld = h;
    e.seg[0].ptr = d.q;
    e.seg[0].group_stride = 0;
    e.seg[1].ptr = page;
    e.seg[1].group_stride = 2 * bh;
    e.seg[2].ptr = page + bh;
    e.seg[2].group_stride = 2 * bh;
    e.scale = 1.f;
    KV_TRY(kvpr_linear(x_slot, h, Lw.wqkv, h, b, 3 * h, h, &e, 0, cs));
  }
  KV_TRY(ck(cudaEventRecord(D.ev_qkv[x.r], cs), "record qkv"));
  if (own_qkv || !(d.zero_copy & 2)) {
    KV_TRY(ck(cudaStreamWaitEvent(ds, D.ev_qkv[x.r], 0), "d2h wait"));
    // the new X row and K,V page, two DMAs in one call (store_activation + store_cache)
    void* dsts[2] = {static_cast<char*>(Lw.host_kv) + static_cast<size_t>(x.s - 1) * 2 * row,
                     d.x_resident ? nullptr : static_cast<char*>(Lw.host_x) + static_cast<size_t>(x.s - 1) * row};
    const void* srcs[2] = {page, x_slot};
    const size_t sizes[2] = {2 * row, d.x_resident ? 0 : row};
    KV_TRY(copy_batch(dsts, srcs, sizes, 2, ds));
    KV_TRY(ck(cudaEventRecord(D.ev_d2h[x.r], ds), "record d2h"));
  } else {  // the previous layer's tail wrote this unit's X row and k, v page into the host stores
    KV_TRY(ck(cudaEventRecord(D.ev_d2h[x.r], cs), "record d2h"));
  }
  // K1 per landed chunk (one launch when X is resident); on its own stream it was issued a unit
  // ahead (issue_k1) and only its completion gates K2
  if (d.recompute_stream == nullptr) {
    KV_TRY(issue_k1_on(D, x, xd, kvd, cs));
  } else {
    KV_TRY(ck(cudaStreamWaitEvent(cs, D.ev_k1[x.r], 0), "wait K1"));
  }
  KV_TRY(ck(cudaStreamWaitEvent(cs, D.ev_kv[x.r], 0), "wait KV"));
  if (d.fused_tail) return fused_tail(D, u, x, kvd, cs);
  KTime t2;
  KV_TRY(kt_begin(D, 1, 2.0 * b * x.s * static_cast<double>(h) * 2, cs, &t2));
  KV_TRY(decode_attention(static_cast<const __half*>(d.q), kvd, static_cast<__half*>(d.attn),
                          static_cast<float*>(d.ws), d.ws_bytes, b, d.heads, h / d.heads, x.s,
                          static_cast<float>(1.0 / sqrt(static_cast<double>(h / d.heads))), cs));
  KV_TRY(kt_end(D, &t2, cs));
  {
    kvpr_epilogue e = simple_epi(d.hres, h, b, h, Lw.bo, KVPR_EPI_F32 | KVPR_EPI_ACCUM);
    KV_TRY(kvpr_linear_ws(d.attn, h, Lw.wo, h, b, h, h, &e, 0, d.ws, d.ws_bytes, cs));
  }
  {
    // LN2 + fc1 + ReLU: one launch on the CUDA-core decode path (batch <= 8), else LN then GEMM
    kvpr_epilogue e = simple_epi(d.mid, d.ffn, b, d.ffn, Lw.b1, KVPR_EPI_RELU);
    KV_TRY(kvpr_layernorm_linear_ws(d.hres, h, Lw.ln2_g, Lw.ln2_b, d.eps, d.y, h, Lw.w1, h, b, d.ffn, h, &e, 0, d.ws,
                                    d.ws_bytes, cs));
  }
  {
    kvpr_epilogue e = simple_epi(d.hres, h, b, h, Lw.b2, KVPR_EPI_F32 | KVPR_EPI_ACCUM);
    KV_TRY(kvpr_linear_ws(d.mid, d.ffn, Lw.w2, d.ffn, b, h, d.ffn, &e, 0, d.ws, d.ws_bytes, cs));
  }
  return ck(cudaEventRecord(D.ev_done[x.r], cs), "record done");
}

}  // namespace

}  // namespace kvpr

using namespace kvpr;

extern "C" {

int kvpr_decoder_create(const kvpr_decoder_desc* desc, const kvpr_layer_desc* layers, void** handle) {
  if (desc == nullptr || layers == nullptr || handle == nullptr || desc->layers <= 0 || desc->batch <= 0 ||
      desc->hidden <= 0 || desc->heads <= 0 || desc->nbuf < 2 || desc->chunks < 1 || desc->chunks > 16) {
    set_error("decoder_create: invalid descriptor (need layers, batch, hidden, heads > 0, nbuf >= 2, 1 <= chunks <= 16)");
    return KVPR_EINVAL;
  }
  Decoder* D = new Decoder();
  D->d = *desc;
  D->layer.assign(layers, layers + desc->layers);
  D->R = desc->layers + desc->nbuf + 2;
  // DMA grouping (kvpr_decoder_desc.dma_group): only where every precondition holds, else per layer
  {
    const int G = desc->dma_group, L = desc->layers;
    bool ok = G > 1 && L % G == 0 && L >= 2 * G && desc->nbuf >= 2 * G && desc->nbuf % G == 0;
    if (ok) {
      D->host_kv_pitch = static_cast<const char*>(layers[1].host_kv) - static_cast<const char*>(layers[0].host_kv);
      const long long row = static_cast<long long>(desc->batch) * desc->hidden * 2;
      ok = D->host_kv_pitch >= 2 * row * desc->capacity;
      for (int j = 1; ok && j < L; ++j)
        ok = static_cast<const char*>(layers[j].host_kv) - static_cast<const char*>(layers[j - 1].host_kv) ==
             D->host_kv_pitch;
    }
    D->group = ok ? G : 1;
  }
  auto mk = [](std::vector<cudaEvent_t>& v, int n) {
    v.resize(n);
    for (auto& e : v)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return false;
    return true;
  };
  if (!mk(D->ev_x, D->R * desc->chunks) || !mk(D->ev_kv, D->R) || !mk(D->ev_qkv, D->R) || !mk(D->ev_d2h, D->R) ||
      !mk(D->ev_done, D->R) || !mk(D->ev_k1, D->R)) {
    set_error("decoder_create: cudaEventCreate failed");
    delete D;
    return KVPR_ECUDA;
  }
  *handle = D;
  return KVPR_OK;
}

int kvpr_decoder_set_timing(void* handle, int enable) {
  Decoder* D = static_cast<Decoder*>(handle);
  if (D == nullptr) return KVPR_EINVAL;
  D->kt.clear();  // pooled events are reused by the next timed run
  D->layer_marks.clear();
  D->step_marks.clear();
  D->t0 = nullptr;
  D->pool_used = 0;
  D->timing = enable != 0;
  return KVPR_OK;
}

int kvpr_decoder_kernel_stats(void* handle, int kind, int* launches, double* mean_seconds, double* mean_units) {
  Decoder* D = static_cast<Decoder*>(handle);
  if (D == nullptr || launches == nullptr || mean_seconds == nullptr || mean_units == nullptr) return KVPR_EINVAL;
  int n = 0;
  double t = 0.0, u = 0.0;
  for (auto& k : D->kt) {
    if (k.kind != kind) continue;
    float ms = 0.f;
    if (cudaEventSynchronize(k.b) != cudaSuccess || cudaEventElapsedTime(&ms, k.a, k.b) != cudaSuccess) {
      set_error("kernel_stats: event query failed");
      return KVPR_ECUDA;
    }
    ++n;
    t += ms * 1e-3;
    u += k.units;
  }
  *launches = n;
  *mean_seconds = n ? t / n : 0.0;
  *mean_units = n ? u / n : 0.0;
  return KVPR_OK;
}

int kvpr_decoder_timeline(void* handle, float* layer_ms, int layer_cap, float* step_ms, int step_cap) {
  Decoder* D = static_cast<Decoder*>(handle);
  if (D == nullptr || (layer_cap > 0 && layer_ms == nullptr) || (step_cap > 0 && step_ms == nullptr)) {
    set_error("decoder_timeline: null handle or output");
    return -KVPR_EINVAL;
  }
  if (D->t0 == nullptr) return 0;
  const int L = D->d.layers;
  const int steps = static_cast<int>(D->step_marks.size());
  if (static_cast<int>(D->layer_marks.size()) != steps * L || layer_cap < steps * L || step_cap < steps) {
    set_error("decoder_timeline: %d steps x %d layers do not fit (caps %d, %d)", steps, L, layer_cap, step_cap);
    return -KVPR_EINVAL;
  }
  auto el = [](cudaEvent_t a, cudaEvent_t b, float* out) {
    return cudaEventSynchronize(b) == cudaSuccess && cudaEventElapsedTime(out, a, b) == cudaSuccess;
  };
  cudaEvent_t prev = D->t0;  // same convention as runtime.KVPRRuntime.decode(timing=...)
  for (int i = 0; i < steps; ++i) {
    if (!el(prev, D->step_marks[i], &step_ms[i])) goto fail;
    prev = D->step_marks[i];
  }
  prev = D->t0;
  for (int i = 0; i < steps; ++i) {
    for (int j = 0; j < L; ++j) {
      if (!el(prev, D->layer_marks[i * L + j], &layer_ms[i * L + j])) goto fail;
      prev = D->layer_marks[i * L + j];
    }
    prev = D->step_marks[i];
  }
  return steps;
fail:
  set_error("decoder_timeline: event query failed");
  return -KVPR_ECUDA;
}

long long kvpr_decoder_launches(void* handle) {
  Decoder* D = static_cast<Decoder*>(handle);
  return D ? D->launches : 0;
}

int kvpr_decoder_destroy(void* handle) {
  Decoder* D = static_cast<Decoder*>(handle);
  if (D == nullptr) return KVPR_OK;
  kvpr_decoder_set_timing(handle, 0);
  for (auto e : D->pool) cudaEventDestroy(e);
  for (auto* v : {&D->ev_x, &D->ev_kv, &D->ev_qkv, &D->ev_d2h, &D->ev_done, &D->ev_k1})
    for (auto e : *v) cudaEventDestroy(e);
  delete D;
  return KVPR_OK;
}

int kvpr_decoder_run(void* handle, int base_len, const int* splits, int steps, int* out_tokens, float* out_logits) {
  clear_error();
  Decoder* D = static_cast<Decoder*>(handle);
  if (D == nullptr || splits == nullptr || steps <= 0) {
    set_error("decoder_run: null handle/splits or steps <= 0");
    return KVPR_EINVAL;
  }
  const kvpr_decoder_desc& d = D->d;
  if (base_len < 1 || base_len + steps > d.capacity) {
    set_error("cache capacity %d exceeded (%d + %d steps)", d.capacity, base_len, steps);
    return KVPR_EINVAL;
  }
  for (int i = 0; i < steps; ++i) {
    if (splits[i] < 0 || splits[i] > base_len + i + 1) {
      set_error("step %d: split %d out of range [0, %d]", i + 1, splits[i], base_len + i + 1);
      return KVPR_EINVAL;
    }
  }
  cudaStream_t cs = static_cast<cudaStream_t>(d.compute_stream);
  const int n = steps * d.layers;
  if (D->timing) {
    D->layer_marks.clear();
    D->step_marks.clear();
    KV_TRY(pool_take(*D, &D->t0));
    KV_TRY(ck(cudaEventRecord(D->t0, cs), "record start"));
  }
  const bool k1_stream = d.recompute_stream != nullptr;
  if (k1_stream) {  // the recompute stream joins the run after everything the caller enqueued on cs
    KV_TRY(ck(cudaEventRecord(D->ev_k1[(D->R - 1) % D->R], cs), "record fork"));
    KV_TRY(ck(cudaStreamWaitEvent(static_cast<cudaStream_t>(d.recompute_stream), D->ev_k1[(D->R - 1) % D->R], 0),
              "fork"));
  }
  KV_TRY(issue_h2d(*D, 0, base_len, splits));
  if (k1_stream) KV_TRY(issue_k1(*D, 0, base_len, splits));
  struct CountLaunches {  // every kernel libkvpr launched during this run (exact, all streams)
    Decoder* D;
    long long start = g_kernel_launches.load();
    ~CountLaunches() { D->launches += g_kernel_launches.load() - start; }
  } counter{D};
  // unit u+1's loads (and its K1) are issued ahead of unit u's compute, except with a single layer:
  // there they wait on unit u's own D2H of the new position (graph.py:286-287), recorded by compute(u)
  const bool ahead = d.layers > 1;
  for (int u = 0; u < n; ++u) {
    if (ahead && u + 1 < n) KV_TRY(issue_h2d(*D, u + 1, base_len, splits));
    if (ahead && u + 1 < n && k1_stream) KV_TRY(issue_k1(*D, u + 1, base_len, splits));
    KV_TRY(compute(*D, u, base_len, splits));
    if (!ahead && u + 1 < n) {
      KV_TRY(issue_h2d(*D, u + 1, base_len, splits));
      if (k1_stream) KV_TRY(issue_k1(*D, u + 1, base_len, splits));
    }
    KV_TRY(mark(*D, D->layer_marks, cs));
    if (u % d.layers == d.layers - 1) {
      const int i = u / d.layers;
      KV_TRY(head(*D, cs));
      if (out_tokens)
        KV_TRY(ck(cudaMemcpyAsync(out_tokens + static_cast<size_t>(i) * d.batch, d.tok, d.batch * sizeof(int),
                                  cudaMemcpyDeviceToDevice, cs),
                  "tokens"));
      if (out_logits)
        KV_TRY(ck(cudaMemcpyAsync(out_logits + static_cast<size_t>(i) * d.batch * d.vocab, d.logits,
                                  static_cast<size_t>(d.batch) * d.vocab * sizeof(float), cudaMemcpyDeviceToDevice,
                                  cs),
                  "logits"));
      KV_TRY(mark(*D, D->step_marks, cs));
    }
  }
  return KVPR_OK;
}

}  // extern "C"
