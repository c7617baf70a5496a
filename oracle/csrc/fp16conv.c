/* IEEE binary16 <-> binary32 conversion for the CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * oracle/opt_ref.py emulates the B200 path's fp16 storage by rounding every materialised tensor
 * through float16 and widening it back (and widens the fp16 host stores every step).  NumPy 2.3's
 * float16 casts are scalar (~2.5 ns/element); at OPT-6.7B width a full-depth teacher-forced decode
 * converts ~9e9 elements per step.  These loops do the same IEEE conversions (exact widening;
 * round-to-nearest-even narrowing, as numpy's astype(float16)) with F16C, split over OpenMP threads.
 * Bit-identical to numpy (tests/test_oracle_cpu.py::test_fp16_helper_matches_numpy). */
#include <immintrin.h>
#include <stddef.h>
#include <stdint.h>
#include <math.h>

void oracle_f16_to_f32(const uint16_t* src, float* dst, size_t n) {
  const size_t n8 = n & ~(size_t)7;
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (size_t i = 0; i < n8; i += 8) {
    __m128i h = _mm_loadu_si128((const __m128i*)(src + i));
    _mm256_storeu_ps(dst + i, _mm256_cvtph_ps(h));
  }
  for (size_t i = n8; i < n; ++i) {
    __m128i h = _mm_cvtsi32_si128(src[i]);
    dst[i] = _mm_cvtss_f32(_mm_cvtph_ps(h));
  }
}

void oracle_f32_to_f16(const float* src, uint16_t* dst, size_t n) {
  const size_t n8 = n & ~(size_t)7;
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (size_t i = 0; i < n8; i += 8) {
    __m256 f = _mm256_loadu_ps(src + i);
    _mm_storeu_si128((__m128i*)(dst + i), _mm256_cvtps_ph(f, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC));
  }
  for (size_t i = n8; i < n; ++i) {
    __m128 f = _mm_set_ss(src[i]);
    dst[i] = (uint16_t)_mm_extract_epi16(_mm_cvtps_ph(f, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC), 0);
  }
}

/* round trip in place: x = float(half(x)) */
void oracle_f32_round_f16(float* x, size_t n) {
  const size_t n8 = n & ~(size_t)7;
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (size_t i = 0; i < n8; i += 8) {
    __m256 f = _mm256_loadu_ps(x + i);
    _mm256_storeu_ps(x + i, _mm256_cvtph_ps(_mm256_cvtps_ph(f, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC)));
  }
  for (size_t i = n8; i < n; ++i) {
    __m128 f = _mm_set_ss(x[i]);
    x[i] = _mm_cvtss_f32(_mm_cvtph_ps(_mm_cvtps_ph(f, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC)));
  }
}

/* Per-head decode attention over a merged cache for the CPU oracle (numerics.py:159-191:
 * softmax(K q / sqrt(d)) V per head with the max subtracted), double accumulation.
 * Positions [0, n32) come from `kv32` (fp32, the rebuilt prefix: K of (p, b) at p*s32_pos + b*s32_b,
 * V s32_v further), [n32, n32 + n16) from `kv16` (fp16 host-store rows from position n32 on, page layout
 * [pos][K|V][batch][hidden]), position n32 + n16 from knew / vnew.  q, knew, vnew, out: [batch][hidden].
 * Work item = one sequence x a group of <= 8 heads, walking positions outermost so each position
 * reads one contiguous run of the row. */

static inline void load16(const uint16_t* src, float* dst, int d) {
  for (int i = 0; i < d; i += 8)
    _mm256_storeu_ps(dst + i, _mm256_cvtph_ps(_mm_loadu_si128((const __m128i*)(src + i))));
}

void oracle_decode_attention(const float* kv32, long n32, long s32_pos, long s32_b, long s32_v, const uint16_t* kv16,
                             long n16, const float* knew, const float* vnew, const float* q, float* out, int batch,
                             int heads, int d, double scale, double* scratch /* batch*heads*(n32+n16+1) */) {
  const long S = n32 + n16 + 1;
  const long hid = (long)heads * d;
  const long row = 2L * batch * hid;  /* elements per position */
  const int G = 8;
  const int groups = (heads + G - 1) / G;
#pragma omp parallel for schedule(dynamic, 1)
  for (long task = 0; task < (long)batch * groups; ++task) {
    const long bi = task / groups;
    const int h0 = (int)(task % groups) * G, h1 = h0 + G < heads ? h0 + G : heads;
    const long off0 = bi * hid + (long)h0 * d, len = (long)(h1 - h0) * d;
    float buf[8 * 256];
    double mx[8], den[8], o[8 * 256];
    for (int g = 0; g < h1 - h0; ++g) mx[g] = -1e300;
    for (long p = 0; p < S; ++p) {
      const float* k;
      if (p < n32) k = kv32 + p * s32_pos + bi * s32_b + (long)h0 * d;
      else if (p < n32 + n16) { load16(kv16 + (p - n32) * row + off0, buf, (int)len); k = buf; }
      else k = knew + off0;
      for (int g = 0; g < h1 - h0; ++g) {
        const float* kk = k + g * d;
        const float* qq = q + off0 + g * d;
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  /* 8 lanes (d % 8 == 0), summed in a fixed order */
        for (int i = 0; i < d; i += 8)
          for (int t = 0; t < 8; ++t) acc[t] += (double)kk[i + t] * qq[i + t];
        const double sv = (((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))) * scale;
        scratch[((bi * heads) + h0 + g) * S + p] = sv;
        if (sv > mx[g]) mx[g] = sv;
      }
    }
    for (int g = 0; g < h1 - h0; ++g) {
      double* sc = scratch + ((bi * heads) + h0 + g) * S;
      double sum = 0.0;
      for (long p = 0; p < S; ++p) {
        sc[p] = exp(sc[p] - mx[g]);
        sum += sc[p];
      }
      den[g] = sum;
    }
    for (long i = 0; i < len; ++i) o[i] = 0.0;
    for (long p = 0; p < S; ++p) {
      const float* v;
      if (p < n32) v = kv32 + p * s32_pos + bi * s32_b + s32_v + (long)h0 * d;
      else if (p < n32 + n16) { load16(kv16 + (p - n32) * row + (long)batch * hid + off0, buf, (int)len); v = buf; }
      else v = vnew + off0;
      for (int g = 0; g < h1 - h0; ++g) {
        const double w = scratch[((bi * heads) + h0 + g) * S + p];
        for (int i = 0; i < d; ++i) o[g * d + i] += w * v[g * d + i];
      }
    }
    for (int g = 0; g < h1 - h0; ++g)
      for (int i = 0; i < d; ++i) out[off0 + g * d + i] = (float)(o[g * d + i] / den[g]);
  }
}
