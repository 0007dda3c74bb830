/* TEST INFRASTRUCTURE ONLY — see flute_oracle.h for the contract.
 *
 * Plain-C restatement of the reference (flutesim) hot path.  Each function
 * cites the reference file:line it restates.  Nothing in the product links
 * this file.
 */
#include "flute_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* binary16 — half.hpp:24-93.  RNE narrowing, exact widening, quiet NaNs.    */
/* ------------------------------------------------------------------------ */

/* Round v / 2^sh to nearest, ties to even (sh >= 1). */
static uint32_t rne_shift(uint32_t v, int sh) {
  if (sh >= 32) return 0;
  uint32_t q = v >> sh;
  uint32_t rem = v & ((1u << sh) - 1u);
  uint32_t half = 1u << (sh - 1);
  if (rem > half || (rem == half && (q & 1u))) q++;
  return q;
}

uint16_t orc_f32_to_f16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint16_t s = (uint16_t)((u >> 16) & 0x8000u);
  const uint32_t a = u & 0x7FFFFFFFu;
  if (a > 0x7F800000u) return (uint16_t)(s | 0x7E00u | ((a & 0x7FFFFFu) >> 13)); /* NaN */
  if (a == 0x7F800000u) return (uint16_t)(s | 0x7C00u);
  const int biased = (int)(a >> 23);
  if (biased == 0) return s; /* f32 zero / subnormal: far below 2^-25 */
  const uint32_t sig = (a & 0x7FFFFFu) | 0x800000u;
  const int e = biased - 127;
  if (e >= -14) {
    const uint32_t r = rne_shift(sig, 13); /* in [1024, 2048] */
    const uint32_t h = ((uint32_t)(e + 15) << 10) + (r - 1024u);
    return (uint16_t)(s | (h >= 0x7C00u ? 0x7C00u : h));
  }
  /* Half subnormal: quantum 2^-24; a carry to 1024 encodes the min normal. */
  return (uint16_t)(s | rne_shift(sig, 13 + (-14 - e)));
}

float orc_f16_to_f32(uint16_t h) {
  const uint32_t s = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu;
  const uint32_t m = h & 0x3FFu;
  uint32_t u;
  if (e == 0x1Fu) {
    u = s | 0x7F800000u | (m << 13);
  } else if (e == 0) {
    const float f = (float)m * 5.9604644775390625e-08f; /* m * 2^-24, exact */
    memcpy(&u, &f, 4);
    u |= s;
  } else {
    u = s | ((e + 112u) << 23) | (m << 13);
  }
  float out;
  memcpy(&out, &u, 4);
  return out;
}

uint16_t orc_f16_add(uint16_t a, uint16_t b) {
  return orc_f32_to_f16(orc_f16_to_f32(a) + orc_f16_to_f32(b));
}

/* ------------------------------------------------------------------------ */
/* NormalFloat table — nf_table.cpp:18-114 (Acklam's published rational     */
/* approximation on the upper half, two Halley steps via erfc, antisymmetric */
/* extension, evenly spaced probability grid, normalisation by q_max).       */
/* ------------------------------------------------------------------------ */

static double acklam_hi(double p) {
  static const double A[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                              -2.759285104469687e+02, 1.383577518672690e+02,
                              -3.066479806614716e+01, 2.506628277459239e+00};
  static const double B[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                              -1.556989798598866e+02, 6.680131188771972e+01,
                              -1.328068155288572e+01};
  static const double C[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                              -2.400758277161838e+00, -2.549732539343734e+00,
                              4.374664141464968e+00, 2.938163982698783e+00};
  static const double D[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                              2.445134137142996e+00, 3.754408661907416e+00};
  if (p <= 1.0 - 0.02425) {
    const double q = p - 0.5, r = q * q;
    const double num = (((((A[0] * r + A[1]) * r + A[2]) * r + A[3]) * r + A[4]) * r + A[5]) * q;
    const double den = ((((B[0] * r + B[1]) * r + B[2]) * r + B[3]) * r + B[4]) * r + 1.0;
    return num / den;
  }
  const double q = sqrt(-2.0 * log(1.0 - p));
  const double num = (((((C[0] * q + C[1]) * q + C[2]) * q + C[3]) * q + C[4]) * q + C[5]);
  const double den = ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
  return -num / den;
}

static double halley(double x, double p) {
  const double e = 0.5 * erfc(-x / 1.4142135623730951) - p;
  const double u = e * 2.5066282746310002 * exp(0.5 * x * x);
  return x - u / (1.0 + 0.5 * x * u);
}

double orc_inverse_normal_cdf(double p) {
  if (!(p > 0.0 && p < 1.0)) return NAN;
  if (p == 0.5) return 0.0;
  if (p < 0.5) return -orc_inverse_normal_cdf(1.0 - p);
  double x = acklam_hi(p);
  x = halley(x, p);
  return halley(x, p);
}

#define ORC_NF_DELTA (0.5 * (1.0 / 30.0 + 1.0 / 32.0))

/* raw NF quantiles Phi^-1(p_i) (nf_table.cpp:75-93) */
int orc_nf_quantiles(int bits, double* q) {
  if (bits < 2 || bits > 4) return 1;
  const double delta = ORC_NF_DELTA;
  const int half = 1 << (bits - 1), cnt = 1 << bits;
  double p[16];
  p[0] = delta;
  p[half - 1] = 0.5;
  p[cnt - 1] = 1.0 - delta;
  for (int i = 1; i < half - 1; ++i) p[i] = delta + (0.5 - delta) * i / (half - 1);
  for (int j = 1; j < half; ++j) p[half - 1 + j] = 0.5 + (0.5 - delta) * j / half;
  for (int i = 0; i < cnt; ++i) q[i] = orc_inverse_normal_cdf(p[i]);
  return 0;
}

/* sigma of the NF grid (nf_table.cpp:71-73) */
double orc_nf_sigma(void) { return 1.0 / orc_inverse_normal_cdf(1.0 - ORC_NF_DELTA); }

int orc_nf_table(int bits, float* values_out) {
  double q[16];
  if (orc_nf_quantiles(bits, q)) return 1;
  const int cnt = 1 << bits;
  for (int i = 0; i < cnt; ++i) values_out[i] = (float)(q[i] / q[cnt - 1]);
  for (int i = 1; i < cnt; ++i)
    if (!(values_out[i - 1] < values_out[i])) return 3;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Quantizer — quantize.cpp:65-128.                                          */
/* ------------------------------------------------------------------------ */

static int cfg_ok(int bits, int group, int k) {
  if (bits < 2 || bits > 4) return 0;
  if (group < 32 || group > 256 || (group & (group - 1)) != 0) return 0;
  if (k >= 0 && k % group != 0) return 0;
  return 1;
}

/* lower_bound neighbours, ties to the smaller index (quantize.cpp:16-26). */
static int nearest(const float* v, int cnt, float r) {
  int lo = 0, hi = cnt; /* first index with v[idx] >= r */
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (v[mid] < r) lo = mid + 1; else hi = mid;
  }
  if (lo == 0) return 0;
  if (lo == cnt) return cnt - 1;
  const float d_lo = r - v[lo - 1];
  const float d_hi = v[lo] - r;
  return d_hi < d_lo ? lo : lo - 1;
}

int orc_quantize(const float* w, int k, int n, int bits, int group, uint8_t* idx_out,
                 uint16_t* scales_out) {
  if (!cfg_ok(bits, group, k)) return 1;
  float table[16];
  int rc = orc_nf_table(bits, table);
  if (rc) return rc;
  const int gpc = k / group, cnt = 1 << bits, zero_idx = (1 << (bits - 1)) - 1;
  const long groups = (long)gpc * n;
  float* absmax = (float*)calloc((size_t)groups, sizeof(float));
  for (long t = 0; t < (long)k * n; ++t)
    if (!isfinite(w[t])) { free(absmax); return 2; }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j) {
      const float a = fabsf(w[(size_t)i * n + j]);
      float* s = &absmax[(size_t)j * gpc + i / group];
      if (a > *s) *s = a;
    }
  for (long g = 0; g < groups; ++g) {
    const uint16_t h = orc_f32_to_f16(absmax[g]);
    if ((h & 0x7C00u) == 0x7C00u) { free(absmax); return 2; }
    scales_out[g] = h;
  }
#pragma omp parallel for schedule(static)
  for (long g = 0; g < groups; ++g) {
    const int j = (int)(g / gpc), i0 = (int)(g % gpc) * group;
    const float s = absmax[g];
    for (int i = i0; i < i0 + group; ++i)
      idx_out[(size_t)i * n + j] =
          (uint8_t)(s == 0.0f ? zero_idx : nearest(table, cnt, w[(size_t)i * n + j] / s));
  }
  free(absmax);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Canonical packer — pack.cpp:18-173.                                       */
/* ------------------------------------------------------------------------ */

int orc_layout_validate(const int* L) {
  for (int t = 0; t < 6; ++t) if (L[t] <= 0) return 1;
  if (L[0] % L[3] || L[1] % L[4] || L[2] % L[5]) return 1;
  if (L[5] % 2) return 1;
  if (((long)L[2] * L[1]) % 32) return 1;
  return 0;
}

int64_t orc_packed_pos(const int* L, int k, int n, int i, int j) {
  (void)n;
  const int64_t tiles_k = k / L[2];
  const int64_t tile = (int64_t)(j / L[1]) * tiles_k + i / L[2];
  const int ki = i % L[2], nj = j % L[1];
  const int64_t frag = (int64_t)(ki / L[5]) * (L[1] / L[4]) + nj / L[4];
  const int64_t within = (int64_t)(ki % L[5]) * L[4] + nj % L[4];
  return tile * ((int64_t)L[2] * L[1]) + frag * ((int64_t)L[5] * L[4]) + within;
}

void orc_unpacked_coords(const int* L, int k, int n, int64_t pos, int* i, int* j) {
  (void)n;
  const int64_t tiles_k = k / L[2];
  const int64_t te = (int64_t)L[2] * L[1], fe = (int64_t)L[5] * L[4];
  const int64_t tile = pos / te, frag = (pos % te) / fe, w = pos % fe;
  const int64_t nfr = L[1] / L[4];
  *i = (int)((tile % tiles_k) * L[2] + (frag / nfr) * L[5] + w / L[4]);
  *j = (int)((tile / tiles_k) * L[1] + (frag % nfr) * L[4] + w % L[4]);
}

int64_t orc_slice_words(int k, int n, int slice_bits) {
  return ((int64_t)k * n * slice_bits + 31) / 32;
}

static void put_bits(uint32_t* words, int64_t pos, int w, uint32_t v) {
  const int64_t bit = pos * w;
  words[bit >> 5] |= v << (bit & 31);
}
static uint32_t get_bits(const uint32_t* words, int64_t pos, int w) {
  const int64_t bit = pos * w;
  return (words[bit >> 5] >> (bit & 31)) & ((1u << w) - 1u);
}

int orc_pack(const uint8_t* idx, int k, int n, int bits, const int* L, uint32_t* s0,
             uint32_t* s1) {
  if (orc_layout_validate(L)) return 1;
  if (k % L[2] || n % L[1]) return 1;
  if (bits < 2 || bits > 4) return 1;
  const int w0 = bits == 3 ? 2 : bits;
  memset(s0, 0, (size_t)orc_slice_words(k, n, w0) * 4);
  if (bits == 3) memset(s1, 0, (size_t)orc_slice_words(k, n, 1) * 4);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j) {
      const uint32_t v = idx[(size_t)i * n + j];
      const int64_t pos = orc_packed_pos(L, k, n, i, j);
      if (bits == 3) {
        put_bits(s0, pos, 2, v >> 1);
        put_bits(s1, pos, 1, v & 1u);
      } else {
        put_bits(s0, pos, bits, v);
      }
    }
  return 0;
}

int orc_unpack(int k, int n, int bits, const int* L, const uint32_t* s0, const uint32_t* s1,
               uint8_t* idx_out) {
  if (orc_layout_validate(L)) return 1;
  const int64_t total = (int64_t)k * n;
  for (int64_t pos = 0; pos < total; ++pos) {
    int i, j;
    orc_unpacked_coords(L, k, n, pos, &i, &j);
    const uint32_t v = bits == 3 ? ((get_bits(s0, pos, 2) << 1) | get_bits(s1, pos, 1))
                                 : get_bits(s0, pos, bits);
    idx_out[(size_t)i * n + j] = (uint8_t)v;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Vectorized LUT — vec_lut.cpp:10-48.                                       */
/* ------------------------------------------------------------------------ */

int orc_vlut(const float* values, int bits, int dup, uint32_t* out) {
  if (dup != 1 && dup != 2 && dup != 4 && dup != 8 && dup != 16) return 1;
  const int cnt = 1 << bits;
  for (int i = 0; i < cnt; ++i)
    for (int j = 0; j < cnt; ++j)
      out[(i << bits) | j] = (uint32_t)orc_f32_to_f16(values[i]) |
                             ((uint32_t)orc_f32_to_f16(values[j]) << 16);
  return 0;
}

uint32_t orc_vec_dequantize(uint32_t e, uint16_t scale) {
  const float s = orc_f16_to_f32(scale);
  const uint16_t a = orc_f32_to_f16(s * orc_f16_to_f32((uint16_t)(e & 0xFFFFu)));
  const uint16_t b = orc_f32_to_f16(s * orc_f16_to_f32((uint16_t)(e >> 16)));
  return (uint32_t)a | ((uint32_t)b << 16);
}

/* Batch form for exhaustive checks: out[s * 2^(2b) + p] = vec_dequantize(p, scales[s]). */
int orc_dequant_table(const uint32_t* vlut, int bits, const uint16_t* scales, int n_scales,
                      uint32_t* out) {
  const int np = 1 << (2 * bits);
#pragma omp parallel for schedule(static)
  for (int s = 0; s < n_scales; ++s)
    for (int p = 0; p < np; ++p) out[(size_t)s * np + p] = orc_vec_dequantize(vlut[p], scales[s]);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Stream-K — streamk.cpp:17-58.                                             */
/* ------------------------------------------------------------------------ */

int orc_plan_stream_k(int tm, int tn, int tk, int P, int64_t* ranges, int64_t* fixups,
                      int max_fixups, int* n_fixups, int64_t* total_slots) {
  if (tm < 1 || tn < 1 || tk < 1 || P < 1) return 1;
  const int64_t U = (int64_t)tm * tn * tk;
  for (int w = 0; w < P; ++w) {
    ranges[2 * w] = U * w / P;
    ranges[2 * w + 1] = U * (w + 1) / P;
  }
  int nf = 0;
  int64_t slots = 0;
  for (int64_t t = 0; t < (int64_t)tm * tn; ++t) {
    const int64_t first = t * tk, last = first + tk - 1;
    int lo = -1, hi = -1, count = 0;
    for (int w = 0; w < P; ++w) {
      const int64_t b = ranges[2 * w], e = ranges[2 * w + 1];
      if (e > b && b <= last && e > first) {
        if (lo < 0) lo = w;
        hi = w;
        ++count;
      }
    }
    if (count <= 1) continue;
    if (fixups && nf < max_fixups) {
      fixups[4 * nf] = t;
      fixups[4 * nf + 1] = hi;
      fixups[4 * nf + 2] = slots;
      fixups[4 * nf + 3] = count - 1;
    }
    slots += count - 1;
    ++nf;
  }
  *n_fixups = nf;
  *total_slots = slots;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Engine — engine.cpp:59-373, serial restatement.                           */
/*                                                                           */
/* Within a worker, accumulation for one output element walks k ascending    */
/* through its units (compute_unit's kf loop, then mma_fragment's kk loop,    */
/* engine.cpp:224-275 / mma.cpp:20-26), a sequential binary32 sum of exact    */
/* f16*f16 products.  At end_of_output_tile the accumulator rounds to f16     */
/* once (engine.cpp:207-209); split tiles reduce contributors' f16 partials  */
/* in ascending order, then the finisher's own (engine.cpp:306-317).          */
/* ------------------------------------------------------------------------ */

typedef struct {
  int m, k, n, bits, group, tile_m;
  const int* L;
  int tiles_m, tiles_n, tiles_k;
} shape_t;

static int make_shape(shape_t* s, int m, int k, int n, int bits, int group, const int* L,
                      int workers, int stages, int tile_m) {
  if (orc_layout_validate(L)) return 1;
  if (!cfg_ok(bits, group, k)) return 1;
  s->m = m; s->k = k; s->n = n; s->bits = bits; s->group = group; s->L = L;
  s->tile_m = tile_m > 0 ? tile_m : L[0];
  if (m < 1 || workers < 1 || stages < 1) return 1;
  if (s->tile_m % L[3]) return 1;
  if (k % L[2] || n % L[1]) return 1;
  s->tiles_m = (m + s->tile_m - 1) / s->tile_m;
  s->tiles_n = n / L[1];
  s->tiles_k = k / L[2];
  return 0;
}

static int real_rows(const shape_t* s, int64_t mt) {
  const int64_t r = (int64_t)s->m - mt * s->tile_m;
  return (int)(r < s->tile_m ? r : s->tile_m);
}

/* Traffic of engine.cpp:87-130 (+ epilogue counters 284-332, 398-417). */
static void count_traffic(const shape_t* s, int P, uint64_t* st) {
  const int* L = s->L;
  const int64_t U = (int64_t)s->tiles_m * s->tiles_n * s->tiles_k;
  const uint64_t tile_bytes = (uint64_t)s->tile_m * L[1] * 2;
  const uint64_t unit_flops = (uint64_t)(s->tile_m / L[3]) * (L[1] / L[4]) * (L[2] / L[5]) *
                              2ull * L[3] * L[4] * L[5];
  memset(st, 0, 7 * sizeof(uint64_t));
  for (int w = 0; w < P; ++w) {
    const int64_t b = U * w / P, e = U * (w + 1) / P;
    if (e <= b) continue;
    st[2] += (uint64_t)(1u << (2 * s->bits)) * 4u;
    for (int64_t u = b; u < e; ++u) {
      const int64_t tile = u / s->tiles_k, mt = tile / s->tiles_n, kt = u % s->tiles_k;
      st[3] += (uint64_t)real_rows(s, mt) * L[2] * 2;
      st[0] += (uint64_t)((int64_t)L[2] * L[1] * s->bits / 8);
      const int64_t k0 = kt * L[2], k1 = k0 + L[2] - 1;
      st[1] += (uint64_t)((k1 / s->group - k0 / s->group + 1) * L[1]) * 2;
      st[6] += unit_flops;
      const int end_tile = (u + 1 >= e) || ((u + 1) / s->tiles_k != tile);
      if (!end_tile) continue;
      const int finished = e > tile * s->tiles_k + s->tiles_k - 1;
      const int started = b <= tile * s->tiles_k;
      if (!finished) { st[4] += tile_bytes; continue; }
      if (!started) {
        int touching = 0;
        for (int v = 0; v < P; ++v) {
          const int64_t vb = U * v / P, ve = U * (v + 1) / P;
          if (ve > vb && vb < (tile + 1) * s->tiles_k && ve > tile * s->tiles_k) ++touching;
        }
        st[4] += tile_bytes * (uint64_t)(touching - 1);
      }
      st[5] += (uint64_t)real_rows(s, mt) * L[1] * 2;
    }
  }
}

int orc_plan_traffic(int m, int k, int n, int bits, int group, const int* L, int workers,
                     int stages, int tile_m, uint64_t* st) {
  shape_t s;
  const int rc = make_shape(&s, m, k, n, bits, group, L, workers, stages, tile_m);
  if (rc) return rc;
  count_traffic(&s, workers, st);
  return 0;
}

/* Dequantized f16 weight (vec_lut.cpp:33-48): f16(f32(s) * f32(f16(T[idx]))). */
static uint16_t deq(uint8_t idx, uint16_t scale, const float* table) {
  return orc_f32_to_f16(orc_f16_to_f32(scale) * orc_f16_to_f32(orc_f32_to_f16(table[idx])));
}

int orc_execute(const uint16_t* x, int m, int k, int n, int bits, int group, const int* L,
                const uint32_t* s0, const uint32_t* s1, const uint16_t* scales,
                const float* table, int P, int stages, int tile_m, uint16_t* y,
                uint64_t* stats) {
  shape_t s;
  const int rc = make_shape(&s, m, k, n, bits, group, L, P, stages, tile_m);
  if (rc) return rc;
  /* Dequantize once: wh[i][j] as binary32 values of the f16 weights. */
  uint8_t* idx = (uint8_t*)malloc((size_t)k * n);
  float* wh = (float*)malloc(sizeof(float) * (size_t)k * n);
  float* xf = (float*)malloc(sizeof(float) * (size_t)m * k);
  if (!idx || !wh || !xf) { free(idx); free(wh); free(xf); return 3; }
  orc_unpack(k, n, bits, L, s0, s1, idx);
  const int gpc = k / group;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j)
      wh[(size_t)i * n + j] =
          orc_f16_to_f32(deq(idx[(size_t)i * n + j], scales[(size_t)j * gpc + i / group], table));
  for (size_t t = 0; t < (size_t)m * k; ++t) xf[t] = orc_f16_to_f32(x[t]);

  const int64_t U = (int64_t)s.tiles_m * s.tiles_n * s.tiles_k;
  const int tn = L[1], tk = L[2], TM = s.tile_m;
  const int64_t out_tiles = (int64_t)s.tiles_m * s.tiles_n;
  /* Partial f16 tiles per (tile, touching worker in ascending order). */
  uint16_t** parts = (uint16_t**)calloc((size_t)out_tiles, sizeof(uint16_t*));
  int* nparts = (int*)calloc((size_t)out_tiles, sizeof(int));
  const size_t tile_elems = (size_t)TM * tn;

  for (int w = 0; w < P; ++w) {
    const int64_t b = U * w / P, e = U * (w + 1) / P;
    int64_t u = b;
    while (u < e) {
      const int64_t tile = u / s.tiles_k;
      const int64_t seg_end = (tile + 1) * s.tiles_k < e ? (tile + 1) * s.tiles_k : e;
      const int64_t mt = tile / s.tiles_n, nt = tile % s.tiles_n;
      const int k0 = (int)((u % s.tiles_k) * tk);
      const int k1 = (int)(((seg_end - 1) % s.tiles_k + 1) * tk);
      uint16_t* y16 = (uint16_t*)calloc(tile_elems, sizeof(uint16_t));
      const int rows = real_rows(&s, mt);
#pragma omp parallel for schedule(static)
      for (int c = 0; c < tn; ++c) {
        const int64_t j = nt * tn + c;
        for (int r = 0; r < TM; ++r) {
          float acc = 0.0f;
          if (r < rows) {
            const float* xr = xf + (size_t)(mt * TM + r) * k;
            for (int i = k0; i < k1; ++i) acc += xr[i] * wh[(size_t)i * n + j];
          }
          y16[(size_t)r * tn + c] = orc_f32_to_f16(acc);
        }
      }
      const int finished = e > tile * s.tiles_k + s.tiles_k - 1;
      const int started = b <= tile * s.tiles_k;
      if (!finished) {
        parts[tile] = (uint16_t*)realloc(parts[tile], tile_elems * 2 * (size_t)(nparts[tile] + 1));
        memcpy(parts[tile] + tile_elems * (size_t)nparts[tile], y16, tile_elems * 2);
        nparts[tile]++;
      } else {
        if (!started) {
          if (nparts[tile] < 1) { free(y16); return 3; }
          for (size_t t = 0; t < tile_elems; ++t) {
            uint16_t sum = parts[tile][t];
            for (int c = 1; c < nparts[tile]; ++c) sum = orc_f16_add(sum, parts[tile][tile_elems * c + t]);
            y16[t] = orc_f16_add(sum, y16[t]);
          }
        }
        for (int r = 0; r < rows; ++r)
          for (int c = 0; c < tn; ++c)
            y[(size_t)(mt * TM + r) * n + nt * tn + c] = y16[(size_t)r * tn + c];
      }
      free(y16);
      u = seg_end;
    }
  }
  for (int64_t t = 0; t < out_tiles; ++t) free(parts[t]);
  free(parts); free(nparts); free(idx); free(wh); free(xf);
  if (stats) count_traffic(&s, P, stats);
  return 0;
}

int orc_reference_f64(const uint16_t* x, int m, int k, int n, int bits, int group,
                      const uint8_t* idx, const uint16_t* scales, const float* table,
                      double* y64) {
  return orc_reference_f64_mode(x, m, k, n, bits, group, idx, scales, table, 1, y64);
}

int orc_reference_f64_mode(const uint16_t* x, int m, int k, int n, int bits, int group,
                           const uint8_t* idx, const uint16_t* scales, const float* table,
                           int f16_weights, double* y64) {
  (void)bits;
  const int gpc = k / group;
  double* wd = (double*)malloc(sizeof(double) * (size_t)k * n);
  if (!wd) return 3;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j)
      wd[(size_t)i * n + j] =
          f16_weights
              ? orc_f16_to_f32(deq(idx[(size_t)i * n + j], scales[(size_t)j * gpc + i / group], table))
              /* dequantize_matrix (quantize.cpp:130-139): binary32 s * T, no f16 rounding */
              : (double)(orc_f16_to_f32(scales[(size_t)j * gpc + i / group]) * table[idx[(size_t)i * n + j]]);
  memset(y64, 0, sizeof(double) * (size_t)m * n);
#pragma omp parallel for schedule(static)
  for (int j0 = 0; j0 < n; j0 += 64) {
    const int j1 = j0 + 64 < n ? j0 + 64 : n;
    for (int r = 0; r < m; ++r)
      for (int i = 0; i < k; ++i) {
        const double xv = orc_f16_to_f32(x[(size_t)r * k + i]);
        if (xv == 0.0) continue;
        const double* wr = wd + (size_t)i * n;
        double* yr = y64 + (size_t)r * n;
        for (int j = j0; j < j1; ++j) yr[j] += xv * wr[j];
      }
  }
  free(wd);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Learned-sigma refinement — quantize.cpp:141-282.  Same loops, same       */
/* binary64 operation order (compiled with -ffp-contract=off).               */
/* ------------------------------------------------------------------------ */

/* 0 ok, 1 config, 2 input (non-finite weight: *bad_i, *bad_j set) */
static int ste_requant(const float* w, int k, int n, int bits, int group, const double* sigma,
                       const double* q, uint8_t* idx, double* what, float* absmax) {
  const int gpc = k / group, cnt = 1 << bits, zero_idx = (1 << (bits - 1)) - 1;
  const long groups = (long)gpc * n;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < k; ++i) {
      const float v = w[(size_t)i * n + j];
      if (!isfinite(v)) return 2;
      float* s = &absmax[(size_t)j * gpc + i / group];
      const float a = fabsf(v);
      if (*s < a) *s = a;
    }
  for (long g = 0; g < groups; ++g) {
    const int j = (int)(g / gpc), i0 = (int)(g % gpc) * group;
    const double eff = (double)absmax[g] * sigma[g];
    double cand[16];
    if (absmax[g] == 0.0f) {
      for (int i = i0; i < i0 + group; ++i) {
        idx[(size_t)i * n + j] = (uint8_t)zero_idx;
        what[(size_t)i * n + j] = 0.0;
      }
      continue;
    }
    for (int c = 0; c < cnt; ++c) cand[c] = eff * q[c];
    for (int i = i0; i < i0 + group; ++i) {
      const double u = (double)w[(size_t)i * n + j];
      int best = 0;
      double bd = fabs(cand[0] - u);
      for (int c = 1; c < cnt; ++c) {
        const double d = fabs(cand[c] - u);
        if (d < bd) { bd = d; best = c; }
      }
      idx[(size_t)i * n + j] = (uint8_t)best;
      what[(size_t)i * n + j] = cand[best];
    }
  }
  return 0;
}

int orc_ste_evaluate(const float* w, const float* x, int m, int k, int n, int bits, int group,
                     const double* sigma, double* loss, double* grad, uint8_t* idx) {
  if (!cfg_ok(bits, group, k)) return 1;
  double q[16];
  orc_nf_quantiles(bits, q);
  const int gpc = k / group;
  const long groups = (long)gpc * n;
  float* absmax = (float*)calloc((size_t)groups, sizeof(float));
  double* what = (double*)malloc(sizeof(double) * (size_t)k * n);
  double* err = (double*)malloc(sizeof(double) * (size_t)m * n);
  int rc = ste_requant(w, k, n, bits, group, sigma, q, idx, what, absmax);
  if (rc == 0) {
#pragma omp parallel for schedule(static)
    for (int t = 0; t < m; ++t)
      for (int j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int i = 0; i < k; ++i)
          acc += (double)x[(size_t)t * k + i] * (what[(size_t)i * n + j] - (double)w[(size_t)i * n + j]);
        err[(size_t)t * n + j] = acc;
      }
    double l = 0.0;
    for (long e = 0; e < (long)m * n; ++e) l += err[e] * err[e];
    *loss = l;
#pragma omp parallel for schedule(static)
    for (long g = 0; g < groups; ++g) {
      const int j = (int)(g / gpc), i0 = (int)(g % gpc) * group;
      double acc = 0.0;
      if (absmax[g] != 0.0f) {
        for (int i = i0; i < i0 + group; ++i) {
          double gij = 0.0;
          for (int t = 0; t < m; ++t) gij += (double)x[(size_t)t * k + i] * err[(size_t)t * n + j];
          acc += 2.0 * gij * (double)absmax[g] * q[idx[(size_t)i * n + j]];
        }
      }
      grad[g] = acc;
    }
  }
  free(absmax);
  free(what);
  free(err);
  return rc;
}

/* 0 ok, 1 config, 2 input, 4 optimization error (*failed_step set) */
int orc_refine_scales(const float* w, const float* x, int m, int k, int n, int bits, int group,
                      int steps, double lr, uint8_t* idx, uint16_t* scales, double* sigma_out,
                      double* losses, int* failed_step) {
  if (steps < 0) return 2;
  int rc = orc_quantize(w, k, n, bits, group, idx, scales);
  if (rc) return rc;
  const long groups = (long)(k / group) * n;
  const double sigma0 = orc_nf_sigma();
  double* sig = sigma_out;
  double* grad = (double*)malloc(sizeof(double) * (size_t)groups);
  uint8_t* tmp = (uint8_t*)malloc((size_t)k * n);
  for (long g = 0; g < groups; ++g) sig[g] = sigma0;
  double l = 0.0;
  if (steps == 0) {
    orc_ste_evaluate(w, x, m, k, n, bits, group, sig, &l, grad, tmp);
    losses[0] = losses[1] = l;
    free(grad);
    free(tmp);
    return 0;
  }
  for (int step = 0; step < steps; ++step) {
    orc_ste_evaluate(w, x, m, k, n, bits, group, sig, &l, grad, tmp);
    if (!isfinite(l)) { *failed_step = step; rc = 4; goto done; }
    if (step == 0) losses[0] = l;
    for (long g = 0; g < groups; ++g) sig[g] -= lr * grad[g];
  }
  orc_ste_evaluate(w, x, m, k, n, bits, group, sig, &l, grad, idx);
  if (!isfinite(l)) { *failed_step = steps; rc = 4; goto done; }
  losses[1] = l;
  {
    const int gpc = k / group;
    for (long g = 0; g < groups; ++g) {
      const int j = (int)(g / gpc), i0 = (int)(g % gpc) * group;
      float am = 0.0f;
      for (int i = i0; i < i0 + group; ++i) {
        const float a = fabsf(w[(size_t)i * n + j]);
        if (am < a) am = a;
      }
      const double folded = (double)am * sig[g] / sigma0;
      if (!(folded >= 0.0) || !isfinite(folded)) { *failed_step = steps; rc = 4; goto done; }
      const uint16_t h = orc_f32_to_f16((float)folded);
      if ((h & 0x7C00u) == 0x7C00u) { *failed_step = steps; rc = 4; goto done; }
      scales[g] = h;
    }
  }
done:
  free(grad);
  free(tmp);
  return rc;
}
