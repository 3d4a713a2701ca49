/*
 * milo_oracle.c — plain-C restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see milo_oracle.h).  Compile with
 * -ffp-contract=off: the reference is compiled for baseline x86-64 (no FMA
 * contraction) and the restatement must reproduce its fp32 rounding bit for bit.
 */
#include "milo_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* binary16 boundary: half.hpp:24-158                                          */
/* ------------------------------------------------------------------------- */

static uint32_t rtne_shift(uint32_t v, int shift) { /* half.hpp:25-33 */
  if (shift <= 0) return v << (-shift);
  if (shift > 31) return 0;
  uint32_t keep = v >> shift;
  uint32_t rem = v & ((1u << shift) - 1u);
  uint32_t halfway = 1u << (shift - 1);
  if (rem > halfway || (rem == halfway && (keep & 1u))) keep += 1;
  return keep;
}

static uint64_t rtne_shift64(uint64_t v, int shift) { /* half.hpp:35-43 */
  if (shift <= 0) return v << (-shift);
  if (shift > 63) return 0;
  uint64_t keep = v >> shift;
  uint64_t rem = v & ((((uint64_t)1) << shift) - 1u);
  uint64_t halfway = ((uint64_t)1) << (shift - 1);
  if (rem > halfway || (rem == halfway && (keep & 1u))) keep += 1;
  return keep;
}

static uint32_t f32_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float bits_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

uint16_t or_float_to_half(float f) { /* half.hpp:47-78 */
  uint32_t x = f32_bits(f);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t exp = (x >> 23) & 0xFFu;
  uint32_t mant = x & 0x7FFFFFu;
  if (exp == 0xFFu) {
    if (mant == 0) return (uint16_t)(sign | 0x7C00u);
    uint32_t m = mant >> 13;
    if (m == 0) m = 1;
    return (uint16_t)(sign | 0x7C00u | m);
  }
  int e = (int)exp - 127 + 15;
  if (e >= 0x1F) return (uint16_t)(sign | 0x7C00u);
  if (e <= 0) {
    int shift = 14 - e;
    if (shift > 31 || exp == 0) return (uint16_t)sign;
    uint32_t full = 0x800000u | mant;
    uint32_t m = rtne_shift(full, shift);
    return (uint16_t)(sign | m);
  }
  uint32_t m = rtne_shift(mant | 0x800000u, 13);
  uint32_t h = (uint32_t)(e << 10) + (m - 0x400u);
  if (h >= 0x7C00u) h = 0x7C00u;
  return (uint16_t)(sign | h);
}

float or_half_to_float(uint16_t h) { /* half.hpp:80-102 */
  uint32_t sign = ((uint32_t)(h & 0x8000u)) << 16;
  uint32_t exp = (h >> 10) & 0x1Fu;
  uint32_t mant = h & 0x3FFu;
  if (exp == 0) {
    if (mant == 0) return bits_f32(sign);
    int shift = 0;
    while (!(mant & 0x400u)) { mant <<= 1; ++shift; }
    mant &= 0x3FFu;
    uint32_t e = (uint32_t)(127 - 14 - shift);
    return bits_f32(sign | (e << 23) | (mant << 13));
  }
  if (exp == 0x1F) return bits_f32(sign | 0x7F800000u | (mant << 13));
  uint32_t e = exp - 15 + 127;
  return bits_f32(sign | (e << 23) | (mant << 13));
}

uint16_t or_double_to_half(double d) { /* half.hpp:105-134 */
  uint64_t x;
  memcpy(&x, &d, 8);
  uint32_t sign = (uint32_t)((x >> 48) & 0x8000u);
  uint32_t exp = (uint32_t)((x >> 52) & 0x7FFu);
  uint64_t mant = x & 0xFFFFFFFFFFFFFull;
  if (exp == 0x7FFu) {
    if (mant == 0) return (uint16_t)(sign | 0x7C00u);
    uint32_t m = (uint32_t)(mant >> 42);
    if (m == 0) m = 1;
    return (uint16_t)(sign | 0x7C00u | m);
  }
  int e = (int)exp - 1023 + 15;
  if (e >= 0x1F) return (uint16_t)(sign | 0x7C00u);
  uint64_t full = (exp == 0) ? mant : (mant | (((uint64_t)1) << 52));
  if (e <= 0) {
    int shift = 43 - e;
    if (shift > 63) return (uint16_t)sign;
    uint64_t m = rtne_shift64(full, shift);
    return (uint16_t)(sign | (uint32_t)m);
  }
  uint64_t m = rtne_shift64(full, 42);
  uint32_t h = (uint32_t)(e << 10) + (uint32_t)(m - 0x400u);
  if (h >= 0x7C00u) h = 0x7C00u;
  return (uint16_t)(sign | h);
}

/* half.hpp:136-158: compute in double, round once */
uint16_t or_half_add(uint16_t a, uint16_t b) {
  return or_double_to_half((double)or_half_to_float(a) + (double)or_half_to_float(b));
}
uint16_t or_half_sub(uint16_t a, uint16_t b) {
  return or_double_to_half((double)or_half_to_float(a) - (double)or_half_to_float(b));
}
uint16_t or_half_mul(uint16_t a, uint16_t b) {
  return or_double_to_half((double)or_half_to_float(a) * (double)or_half_to_float(b));
}
uint16_t or_half_fma(uint16_t a, uint16_t b, uint16_t c) {
  return or_double_to_half(
      fma((double)or_half_to_float(a), (double)or_half_to_float(b), (double)or_half_to_float(c)));
}
static uint16_t half_neg(uint16_t a) { return (uint16_t)(a ^ 0x8000u); }

/* ------------------------------------------------------------------------- */
/* zero-bit-waste INT3 storage: pack.hpp:6-24, pack.cpp:33-302                 */
/* ------------------------------------------------------------------------- */

int or_pack32(const uint8_t* codes, size_t n, uint32_t* w) { /* pack.cpp:33-54 */
  if (n != 32) return OR_SHAPE;
  for (int i = 0; i < 32; ++i)
    if (codes[i] > 7) return OR_RANGE;
  w[0] = w[1] = w[2] = 0;
  for (int j = 0; j < 3; ++j)
    for (int k = 0; k < 8; ++k) w[j] |= (uint32_t)codes[8 * j + k] << (3 * k);
  uint32_t rest = 0;
  for (int k = 0; k < 8; ++k) rest |= (uint32_t)codes[24 + k] << (3 * k);
  for (int j = 0; j < 3; ++j) w[j] |= ((rest >> (8 * j)) & 0xFFu) << 24;
  return OR_OK;
}

void or_unpack32(const uint32_t* w, uint8_t* codes) { /* pack.cpp:56-68 */
  for (int j = 0; j < 3; ++j)
    for (int k = 0; k < 8; ++k) codes[8 * j + k] = (uint8_t)((w[j] >> (3 * k)) & 0x7u);
  uint32_t rest = (w[0] >> 24) | ((w[1] >> 24) << 8) | ((w[2] >> 24) << 16);
  for (int k = 0; k < 8; ++k) codes[24 + k] = (uint8_t)((rest >> (3 * k)) & 0x7u);
}

uint64_t or_tiled_position(uint64_t rows, uint64_t cols, uint64_t i, uint64_t j) {
  (void)rows; /* pack.cpp:133-139 */
  const uint64_t tiles_per_row = cols / 64;
  const uint64_t ti = i / 16, tj = j / 64, r = i % 16, c = j % 64;
  return (ti * tiles_per_row + tj) * (16 * 64) + r * 64 + c;
}

int or_pack_matrix(uint64_t rows, uint64_t cols, const uint8_t* codes, const float* scales,
                   const float* zeros, uint64_t group_size, int tiled, int split,
                   uint32_t* words, uint32_t* plane_a, uint32_t* plane_b, uint16_t* scales_h,
                   uint16_t* zeros_h) {
  /* check_packable pack.cpp:72-76; symmetric extra checks 118-121; tiled 143-145 */
  if (rows == 0 || cols == 0) return OR_SHAPE;
  if (cols % 32 != 0) return OR_SHAPE;
  if (zeros == NULL) {
    if (cols % group_size != 0) return OR_SHAPE;
    if (tiled) return OR_CONFIG; /* reshuffle_tiled takes QuantizedMatrix (asymmetric) */
  }
  if (tiled && (rows % 16 != 0 || cols % 64 != 0)) return OR_SHAPE;
  const uint64_t n = rows * cols;
  uint8_t* stream = (uint8_t*)malloc(n);
  if (tiled) {
    for (uint64_t i = 0; i < rows; ++i)
      for (uint64_t j = 0; j < cols; ++j)
        stream[or_tiled_position(rows, cols, i, j)] = codes[i * cols + j];
  } else {
    memcpy(stream, codes, n);
  }
  const uint64_t groups = n / 32;
  for (uint64_t g = 0; g < groups; ++g) { /* pack_stream pack.cpp:78-87 */
    uint32_t w[3];
    int st = or_pack32(stream + g * 32, 32, w);
    if (st) { free(stream); return st; }
    if (split) { /* split_planes pack.cpp:163-178 */
      plane_a[g * 2 + 0] = w[0];
      plane_a[g * 2 + 1] = w[1];
      plane_b[g] = w[2];
    } else {
      words[g * 3 + 0] = w[0];
      words[g * 3 + 1] = w[1];
      words[g * 3 + 2] = w[2];
    }
  }
  free(stream);
  const uint64_t qg = n / group_size;
  for (uint64_t g = 0; g < qg; ++g) scales_h[g] = or_float_to_half(scales[g]);
  if (zeros && zeros_h)
    for (uint64_t g = 0; g < qg; ++g) zeros_h[g] = or_float_to_half(zeros[g]);
  return OR_OK;
}

static void word3(const uint32_t* words, const uint32_t* pa, const uint32_t* pb, int split,
                  uint64_t g, uint32_t* w) { /* PackedInt3Matrix::word pack.hpp:62-65 */
  if (!split) {
    w[0] = words[g * 3 + 0];
    w[1] = words[g * 3 + 1];
    w[2] = words[g * 3 + 2];
  } else {
    w[0] = pa[g * 2 + 0];
    w[1] = pa[g * 2 + 1];
    w[2] = pb[g];
  }
}

int or_unpack_codes(uint64_t rows, uint64_t cols, int layout, int split, const uint32_t* words,
                    const uint32_t* pa, const uint32_t* pb, uint8_t* out) {
  /* pack.cpp:196-211 */
  const uint64_t n = rows * cols, groups = n / 32;
  uint8_t* stream = (uint8_t*)malloc(n);
  for (uint64_t g = 0; g < groups; ++g) {
    uint32_t w[3];
    word3(words, pa, pb, split, g, w);
    or_unpack32(w, stream + g * 32);
  }
  if (layout == 0) {
    memcpy(out, stream, n);
  } else {
    for (uint64_t i = 0; i < rows; ++i)
      for (uint64_t j = 0; j < cols; ++j)
        out[i * cols + j] = stream[or_tiled_position(rows, cols, i, j)];
  }
  free(stream);
  return OR_OK;
}

void or_fast_dequant_pair(uint32_t word, int pair, int mode, uint16_t* out2) {
  /* pack.cpp:215-234 */
  const uint32_t t = word >> (6 * pair);
  const uint32_t lanes = (t & 0x7u) | ((t << 16) & 0x00380000u) | 0x64006400u;
  const uint16_t lo = (uint16_t)(lanes & 0xFFFFu), hi = (uint16_t)(lanes >> 16);
  if (mode == 0) {
    out2[0] = or_half_sub(lo, 0x6404);
    out2[1] = or_half_fma(hi, 0x3000, 0xD820);
  } else {
    out2[0] = or_half_sub(lo, 0x6400);
    out2[1] = or_half_fma(hi, 0x3000, 0xD800);
  }
}

uint16_t or_symmetric_step(uint16_t s) { /* pack.cpp:236-238 */
  return or_double_to_half((double)or_half_to_float(s) * 2.0 / 7.0);
}
uint16_t or_asymmetric_offset(uint16_t s, uint16_t z) { /* pack.cpp:240-242 */
  return half_neg(or_half_mul(s, z));
}

int or_dequant_packed_half(uint64_t rows, uint64_t cols, int layout, int split,
                           uint64_t group_size, const uint32_t* words, const uint32_t* pa,
                           const uint32_t* pb, const uint16_t* scales, const uint16_t* zeros,
                           int mode, uint16_t* out) {
  /* pack.cpp:244-295 */
  if (mode == 1 && zeros == NULL) return OR_CONFIG;
  const uint64_t n = rows * cols, groups = n / 32;
  uint16_t* stream = (uint16_t*)malloc(n * 2);
  for (uint64_t g = 0; g < groups; ++g) {
    uint32_t w[3];
    word3(words, pa, pb, split, g, w);
    uint16_t* o = stream + g * 32;
    for (int j = 0; j < 3; ++j)
      for (int pair = 0; pair < 4; ++pair) or_fast_dequant_pair(w[j], pair, mode, o + 8 * j + 2 * pair);
    const uint32_t w3 = (w[0] >> 24) | ((w[1] >> 24) << 8) | ((w[2] >> 24) << 16);
    for (int pair = 0; pair < 4; ++pair) or_fast_dequant_pair(w3, pair, mode, o + 24 + 2 * pair);
  }
  if (layout == 0) {
    memcpy(out, stream, n * 2);
  } else {
    for (uint64_t i = 0; i < rows; ++i)
      for (uint64_t j = 0; j < cols; ++j)
        out[i * cols + j] = stream[or_tiled_position(rows, cols, i, j)];
  }
  free(stream);
  const uint64_t qg = n / group_size;
  for (uint64_t g = 0; g < qg; ++g) {
    uint16_t* v = out + g * group_size;
    if (mode == 0) {
      const uint16_t step = or_symmetric_step(scales[g]);
      for (uint64_t k = 0; k < group_size; ++k) v[k] = or_half_mul(v[k], step);
    } else {
      const uint16_t s = scales[g], off = or_asymmetric_offset(s, zeros[g]);
      for (uint64_t k = 0; k < group_size; ++k) v[k] = or_half_fma(v[k], s, off);
    }
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* grouped quantizer: quant.cpp:23-76                                          */
/* ------------------------------------------------------------------------- */

int or_quantize_minmax(uint64_t rows, uint64_t cols, uint64_t gs, const float* w,
                       uint8_t* codes, float* scales, float* zeros) {
  if (rows == 0 || cols == 0) return OR_SHAPE; /* check_grouping quant.cpp:12-17 */
  if (cols % gs != 0) return OR_SHAPE;
  const uint64_t ng = rows * cols / gs;
  const float levels = 7.0f, maxc = 7.0f;
  for (uint64_t g = 0; g < ng; ++g) { /* init_quant_params quant.cpp:23-45 */
    const float* v = w + g * gs;
    float lo = v[0], hi = v[0];
    for (uint64_t k = 1; k < gs; ++k) {
      lo = v[k] < lo ? v[k] : lo; /* std::min(lo, v[k]) */
      hi = hi < v[k] ? v[k] : hi; /* std::max(hi, v[k]) */
    }
    float s = (hi - lo) / levels;
    if (s < 1e-8f) s = 1e-8f;
    scales[g] = s;
    zeros[g] = -lo / s;
    if (!isfinite(scales[g]) || !isfinite(zeros[g])) return OR_NUMERIC;
  }
  for (uint64_t g = 0; g < ng; ++g) { /* quantize quant.cpp:47-76 */
    const float s = scales[g], z = zeros[g];
    for (uint64_t k = 0; k < gs; ++k) {
      float r = roundf(w[g * gs + k] / s + z);
      if (r < 0.0f) r = 0.0f;
      if (r > maxc) r = maxc;
      codes[g * gs + k] = (uint8_t)r;
    }
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* symmetric INT3 compensator factors: lowrank.cpp:19-50,89-134                */
/* ------------------------------------------------------------------------- */

int or_symm_int3_quantize(const float* values, uint64_t rows, uint64_t cols, uint64_t gs,
                          uint8_t* codes, float* scales) {
  if (gs == 0) return OR_SHAPE;
  const uint64_t gpr = (cols + gs - 1) / gs;
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t g = 0; g < gpr; ++g) {
      const uint64_t begin = g * gs, end = begin + gs < cols ? begin + gs : cols;
      float s = 0.0f;
      for (uint64_t j = begin; j < end; ++j) {
        float a = fabsf(values[i * cols + j]);
        s = s < a ? a : s; /* std::max(s, |w|) */
      }
      s = s < 1e-8f ? 1e-8f : s;
      scales[i * gpr + g] = s;
      for (uint64_t j = begin; j < end; ++j) {
        float code = roundf(7.0f * values[i * cols + j] / (2.0f * s)) + 4.0f;
        code = code < 0.0f ? 0.0f : (code > 7.0f ? 7.0f : code);
        codes[i * cols + j] = (uint8_t)code;
      }
    }
  return OR_OK;
}

void or_symm_int3_dequantize(uint64_t rows, uint64_t cols, uint64_t gs, const uint8_t* codes,
                             const float* scales, float* out) {
  const uint64_t gpr = (cols + gs - 1) / gs;
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t j = 0; j < cols; ++j) {
      const float s = scales[i * gpr + j / gs];
      const float step = s * (2.0f / 7.0f);
      out[i * cols + j] = step * ((float)codes[i * cols + j] - 4.0f);
    }
}

/* Compensator::u_real / v_real, lowrank.cpp:19-32 */
static float* comp_u_real(const or_comp* c) {
  float* u = (float*)malloc(c->rows * c->rank * 4 + 4);
  if (c->storage == 0) {
    memcpy(u, c->U, c->rows * c->rank * 4);
  } else {
    or_symm_int3_dequantize(c->rows, c->rank, c->group_size, c->qu_codes, c->qu_scales, u);
  }
  return u;
}

static float* comp_v_real(const or_comp* c) {
  float* v = (float*)malloc(c->rank * c->cols * 4 + 4);
  if (c->storage == 0) {
    memcpy(v, c->V, c->rank * c->cols * 4);
  } else {
    float* vt = (float*)malloc(c->cols * c->rank * 4 + 4);
    or_symm_int3_dequantize(c->cols, c->rank, c->group_size, c->qvt_codes, c->qvt_scales, vt);
    for (uint64_t j = 0; j < c->cols; ++j)
      for (uint64_t k = 0; k < c->rank; ++k) v[k * c->cols + j] = vt[j * c->rank + k];
    free(vt);
  }
  return v;
}

/* Eager fp32 product (a: r x kk, b: kk x c), ascending inner index, separate
 * multiply and add — the arithmetic of the reference's dense products as
 * compiled in oracle/_ref (oracle/ref/eigen_shim). */
static float* product(const float* a, const float* b, uint64_t r, uint64_t kk, uint64_t c) {
  float* o = (float*)calloc(r * c + 1, 4);
  for (uint64_t i = 0; i < r; ++i)
    for (uint64_t q = 0; q < kk; ++q) {
      const float av = a[i * kk + q];
      for (uint64_t j = 0; j < c; ++j) o[i * c + j] += av * b[q * c + j];
    }
  return o;
}

/* ------------------------------------------------------------------------- */
/* W3A16 GEMM: gemm.cpp:15-199                                                  */
/* ------------------------------------------------------------------------- */

int or_gemm_validate(const or_gemm_cfg* cfg) { /* gemm.cpp:23-30 */
  const int tk = cfg->tile_k, tn = cfg->tile_n;
  if (!((tk == 64 && tn == 256) || (tk == 128 && tn == 128) || (tk == 256 && tn == 64)))
    return OR_CONFIG;
  if (cfg->group_size != 64) return OR_CONFIG;
  if (cfg->pipeline_depth < 1) return OR_CONFIG;
  return OR_OK;
}

int or_pipeline_tail_check(uint64_t k, const or_gemm_cfg* cfg, int* stages, int max_stages,
                           int* n_stages) { /* gemm.cpp:32-47 */
  int st = or_gemm_validate(cfg);
  if (st) return st;
  const uint64_t tk = (uint64_t)cfg->tile_k;
  if (k % tk != 0) return OR_SHAPE;
  int remaining = (int)(k / tk), n = 0;
  while (remaining > 0) {
    int s = remaining < cfg->pipeline_depth ? remaining : cfg->pipeline_depth;
    if (n < max_stages) stages[n] = s;
    ++n;
    remaining -= s;
  }
  *n_stages = n;
  return OR_OK;
}

int or_gemm_w3a16(const float* A, uint64_t m0, uint64_t a_cols, const or_packed* W,
                  const or_comp* comp, const or_gemm_cfg* cfg, float* Cout) {
  /* validation order: gemm.cpp:120-139 */
  int st = or_gemm_validate(cfg);
  if (st) return st;
  if (W->group_size != 64) return OR_CONFIG;
  if (cfg->mode != W->mode) return OR_CONFIG;
  if (cfg->mode == 1 && W->zeros == NULL) return OR_CONFIG;
  const uint64_t k = W->rows, n = W->cols;
  const uint64_t tk = (uint64_t)cfg->tile_k, tn = (uint64_t)cfg->tile_n;
  if (k % tk != 0 || n % tn != 0) return OR_SHAPE;
  if (a_cols != k) return OR_SHAPE;
  if (comp && (comp->rows != k || comp->cols != n)) return OR_SHAPE;

  /* pad_batch gemm.cpp:49-60 and binary16 activations gemm.cpp:144-146 */
  const uint64_t m = (m0 + 15) / 16 * 16;
  float* Ah = (float*)calloc(m * k + 1, 4);
  for (uint64_t i = 0; i < m0 * k; ++i) Ah[i] = or_half_to_float(or_float_to_half(A[i]));
  for (uint64_t i = m0 * k; i < m * k; ++i) Ah[i] = or_half_to_float(or_float_to_half(0.0f));

  float* C = (float*)calloc(m * n + 1, 4);
  float* block = (float*)malloc(tk * tn * 4);
  float lut[8];
  for (uint64_t n0 = 0; n0 < n; n0 += tn) {           /* gemm.cpp:153 */
    for (uint64_t k0 = 0; k0 < k; k0 += tk) {           /* stage order = tile order :155-157 */
      /* dequant_block gemm.cpp:88-113 */
      for (uint64_t r = 0; r < tk; ++r) {
        const uint64_t row = k0 + r;
        float* out = block + r * tn;
        for (uint64_t j0 = 0; j0 < tn; j0 += 64) {
          const uint64_t col = n0 + j0;
          const uint64_t qg = (row * n + col) / W->group_size;
          /* GroupLut::build gemm.cpp:70-84 */
          const uint16_t s = W->scales[qg];
          if (W->mode == 0) {
            const uint16_t step = or_symmetric_step(s);
            for (int c = 0; c < 8; ++c)
              lut[c] = or_half_to_float(or_half_mul(or_double_to_half((double)(c - 4)), step));
          } else {
            const uint16_t z = W->zeros ? W->zeros[qg] : 0;
            const uint16_t off = or_asymmetric_offset(s, z);
            for (int c = 0; c < 8; ++c)
              lut[c] = or_half_to_float(or_half_fma(or_double_to_half((double)c), s, off));
          }
          for (uint64_t hb = 0; hb < 2; ++hb) {
            const uint64_t flat = row * n + col + hb * 32;
            const uint64_t pos =
                W->layout == 0 ? flat : or_tiled_position(W->rows, W->cols, row, col + hb * 32);
            uint32_t w[3];
            uint8_t codes[32];
            word3(W->words, W->plane_a, W->plane_b, W->split, pos / 32, w);
            or_unpack32(w, codes);
            float* o = out + j0 + hb * 32;
            for (int c = 0; c < 32; ++c) o[c] = lut[codes[c]];
          }
        }
      }
      /* fp32 accumulation, k ascending, zero activations skipped: gemm.cpp:159-168 */
      for (uint64_t i = 0; i < m; ++i) {
        const float* arow = Ah + i * k + k0;
        float* crow = C + i * n + n0;
        for (uint64_t kk = 0; kk < tk; ++kk) {
          const float a = arow[kk];
          if (a == 0.0f) continue;
          const float* wrow = block + kk * tn;
          for (uint64_t j = 0; j < tn; ++j) crow[j] += a * wrow[j];
        }
      }
    }
  }
  free(block);

  if (comp && comp->rank > 0) { /* gemm.cpp:173-194 */
    float* u = comp_u_real(comp);
    float* v = comp_v_real(comp);
    float* add;
    if (cfg->materialize_compensator) {
      float* uv = product(u, v, k, comp->rank, n); /* compensator_apply lowrank.cpp:136-149 */
      add = product(Ah, uv, m, k, n);
      free(uv);
    } else {
      float* T = product(Ah, u, m, k, comp->rank);
      add = product(T, v, m, comp->rank, n);
      free(T);
    }
    for (uint64_t i = 0; i < m * n; ++i) C[i] += add[i];
    free(add);
    free(u);
    free(v);
  }
  memcpy(Cout, C, m0 * n * 4); /* first m rows: gemm.cpp:196-198 */
  free(C);
  free(Ah);
  return OR_OK;
}

uint64_t or_matrix_memory_bytes(uint64_t rows, uint64_t cols, uint64_t rank, int bits,
                                uint64_t gs, int comp_bits) { /* tensor_store.cpp:247-266 */
  if (rank > (rows < cols ? rows : cols)) return 0;
  if (gs == 0 || cols % gs != 0) return 0;
  const uint64_t n = rows * cols;
  const uint64_t code_bytes = n * (uint64_t)bits / 8;
  const uint64_t meta_bytes = 2 * (n / gs) * 2;
  const uint64_t comp_entries = (rows + cols) * rank;
  const uint64_t comp_code_bytes = comp_entries * (uint64_t)comp_bits / 8;
  const uint64_t comp_groups = rank == 0 ? 0 : (rows + cols) * ((rank + gs - 1) / gs);
  return code_bytes + meta_bytes + comp_code_bytes + comp_groups * 2;
}

/* ------------------------------------------------------------------------- */
/* MoE layer (new, see header)                                                  */
/* ------------------------------------------------------------------------- */

void or_router_gemm(const float* x, uint64_t m, uint64_t d, const uint16_t* gate, int E, float* logits) {
  for (uint64_t t = 0; t < m; ++t)
    for (int e = 0; e < E; ++e) {
      float lane[32];
      for (int l = 0; l < 32; ++l) {
        float acc = 0.0f;
        for (uint64_t k = (uint64_t)l; k < d; k += 32) {
          const float a = or_half_to_float(or_float_to_half(x[t * d + k]));
          const float g = or_half_to_float(gate[(uint64_t)e * d + k]);
          acc = fmaf(a, g, acc);  /* the product is exact: one rounding, like the device FFMA */
        }
        lane[l] = acc;
      }
      for (int off = 16; off > 0; off >>= 1) {
        float nxt[32];
        for (int l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ off];
        memcpy(lane, nxt, sizeof(lane));
      }
      logits[t * (uint64_t)E + (uint64_t)e] = lane[0];
    }
}

void or_router_topk(const float* logits, uint64_t m, int E, int K, int score_mode,
                    int32_t* ids, float* wts) {
  float* p = (float*)malloc((size_t)E * 4);
  for (uint64_t t = 0; t < m; ++t) {
    const float* l = logits + t * (uint64_t)E;
    int32_t* id = ids + t * (uint64_t)K;
    /* selection: k passes, each picks the largest remaining logit, lowest id on ties */
    for (int k = 0; k < K; ++k) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        int used = 0;
        for (int q = 0; q < k; ++q) used |= (id[q] == e);
        if (used) continue;
        if (best < 0 || l[e] > l[best]) best = e;
      }
      id[k] = best;
    }
    float* w = wts + t * (uint64_t)K;
    if (score_mode == 0) {
      const float mx = l[id[0]];
      float sum = 0.0f;
      for (int k = 0; k < K; ++k) { w[k] = expf(l[id[k]] - mx); sum += w[k]; }
      for (int k = 0; k < K; ++k) w[k] = w[k] / sum;
    } else {
      float mx = l[0];
      for (int e = 1; e < E; ++e) mx = l[e] > mx ? l[e] : mx;
      float sum = 0.0f;
      for (int e = 0; e < E; ++e) { p[e] = expf(l[e] - mx); sum += p[e]; }
      for (int k = 0; k < K; ++k) w[k] = p[id[k]] / sum;
    }
  }
  free(p);
}

typedef struct {
  const or_expert* ex;
  const float* x;
  uint64_t d;
  const uint64_t* rows; /* token ids of this expert */
  uint64_t n_rows;
  float* y;             /* n_rows x d */
  int status;
} moe_job;

static void run_expert(moe_job* j) {
  const or_expert* ex = j->ex;
  const uint64_t mr = j->n_rows, d = j->d, f = ex->w[0].cols;
  /* tile shape per matrix: (128, 128) where it divides, else one of the reference's other
     allowed shapes (gemm.cpp:23-30: 64x256, 256x64); the tile only orders the fp32 sums */
  or_gemm_cfg cfg = {128, 128, 64, ex->w[0].mode, 4, 0};
#define PICK_TILE(W)                                                        \
  do {                                                                      \
    const uint64_t kk = (W).rows, nn = (W).cols;                            \
    if (kk % 128 == 0 && nn % 128 == 0) { cfg.tile_k = 128; cfg.tile_n = 128; } \
    else if (kk % 256 == 0 && nn % 64 == 0) { cfg.tile_k = 256; cfg.tile_n = 64; } \
    else if (kk % 64 == 0 && nn % 256 == 0) { cfg.tile_k = 64; cfg.tile_n = 256; } \
  } while (0)
  PICK_TILE(ex->w[0]);
  float* xe = (float*)malloc(mr * d * 4 + 4);
  for (uint64_t i = 0; i < mr; ++i) memcpy(xe + i * d, j->x + j->rows[i] * d, d * 4);
  float* h1 = (float*)malloc(mr * f * 4 + 4);
  float* h3 = (float*)malloc(mr * f * 4 + 4);
  int st = or_gemm_w3a16(xe, mr, d, &ex->w[0], ex->has_comp[0] ? &ex->c[0] : NULL, &cfg, h1);
  cfg.mode = ex->w[1].mode;
  PICK_TILE(ex->w[1]);
  if (!st) st = or_gemm_w3a16(xe, mr, d, &ex->w[1], ex->has_comp[1] ? &ex->c[1] : NULL, &cfg, h3);
  if (!st) {
    for (uint64_t i = 0; i < mr * f; ++i) {
      const float a = h1[i];
      h1[i] = a / (1.0f + expf(-a)) * h3[i];
    }
    cfg.mode = ex->w[2].mode;
    PICK_TILE(ex->w[2]);
    st = or_gemm_w3a16(h1, mr, f, &ex->w[2], ex->has_comp[2] ? &ex->c[2] : NULL, &cfg, j->y);
  }
#undef PICK_TILE
  j->status = st;
  free(xe);
  free(h1);
  free(h3);
}

typedef struct {
  moe_job* jobs;
  int n_jobs;
  int next;
  pthread_mutex_t mu;
} job_queue;

static void* worker(void* arg) {
  job_queue* q = (job_queue*)arg;
  for (;;) {
    pthread_mutex_lock(&q->mu);
    int i = q->next++;
    pthread_mutex_unlock(&q->mu);
    if (i >= q->n_jobs) return NULL;
    run_expert(&q->jobs[i]);
  }
}

int or_moe_forward(const or_expert* experts, int n_experts, const or_expert* shared,
                   int n_shared, const float* x, uint64_t m, uint64_t d, int K,
                   const int32_t* ids, const float* wts, int n_threads, float* out) {
  const int total = n_experts + n_shared;
  moe_job* jobs = (moe_job*)calloc((size_t)total, sizeof(moe_job));
  uint64_t** rows = (uint64_t**)calloc((size_t)total, sizeof(uint64_t*));
  uint64_t* all_rows = (uint64_t*)malloc((m + 1) * 8);
  for (uint64_t t = 0; t < m; ++t) all_rows[t] = t;
  int n_jobs = 0;
  int* job_of = (int*)malloc((size_t)total * sizeof(int));
  for (int e = 0; e < total; ++e) {
    job_of[e] = -1;
    uint64_t cnt = 0;
    if (e < n_experts) {
      rows[e] = (uint64_t*)malloc((m * (uint64_t)K + 1) * 8);
      for (uint64_t t = 0; t < m; ++t)
        for (int k = 0; k < K; ++k)
          if (ids[t * (uint64_t)K + (uint64_t)k] == e) rows[e][cnt++] = t;
    } else {
      cnt = m;
    }
    if (cnt == 0) continue;
    moe_job* j = &jobs[n_jobs];
    j->ex = e < n_experts ? &experts[e] : &shared[e - n_experts];
    j->x = x;
    j->d = d;
    j->rows = e < n_experts ? rows[e] : all_rows;
    j->n_rows = cnt;
    j->y = (float*)malloc(cnt * d * 4 + 4);
    job_of[e] = n_jobs++;
  }
  if (n_threads <= 1 || n_jobs <= 1) {
    for (int i = 0; i < n_jobs; ++i) run_expert(&jobs[i]);
  } else {
    job_queue q = {jobs, n_jobs, 0, PTHREAD_MUTEX_INITIALIZER};
    int nt = n_threads < n_jobs ? n_threads : n_jobs;
    pthread_t* th = (pthread_t*)malloc((size_t)nt * sizeof(pthread_t));
    for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, worker, &q);
    for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
    free(th);
  }
  int st = OR_OK;
  for (int i = 0; i < n_jobs; ++i)
    if (jobs[i].status) st = jobs[i].status;
  if (!st) {
    uint64_t* cursor = (uint64_t*)calloc((size_t)total + 1, 8);
    memset(out, 0, m * d * 4);
    for (uint64_t t = 0; t < m; ++t) {
      for (int k = 0; k < K; ++k) {
        const int e = ids[t * (uint64_t)K + (uint64_t)k];
        if (e < 0 || e >= n_experts) continue;
        const float w = wts[t * (uint64_t)K + (uint64_t)k];
        const float* yr = jobs[job_of[e]].y + (cursor[e]++) * d;
        for (uint64_t c = 0; c < d; ++c) out[t * d + c] += w * yr[c];
      }
      for (int s = 0; s < n_shared; ++s) {
        const float* yr = jobs[job_of[n_experts + s]].y + t * d;
        for (uint64_t c = 0; c < d; ++c) out[t * d + c] += 1.0f * yr[c];
      }
    }
    free(cursor);
  }
  for (int i = 0; i < n_jobs; ++i) free(jobs[i].y);
  for (int e = 0; e < n_experts; ++e) free(rows[e]);
  free(rows);
  free(all_rows);
  free(job_of);
  free(jobs);
  return st;
}
