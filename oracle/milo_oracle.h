/*
 * milo_oracle — CPU restatement of the reference's hot path, in plain C11.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker, never the thing
 * measured or shipped: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product library (libmilo_b200.so) does
 * not link it and has no CPU fallback.
 *
 * Each function restates the reference function named beside it
 * (/root/reference/proj/...:line).  Parity pinning: the restatement is checked
 * bit-for-bit against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py driving oracle/_ref/libmilo_ref.so, the
 * reference sources compiled by oracle/build_ref.sh), see
 * tests/test_oracle_golden.py.  The MoE routing / SwiGLU / combine layer has
 * no reference counterpart and is defined here; its
 * parity is pinned only against ref_moe_forward, the same composition built
 * from the reference's gemm_w3a16.
 *
 * Status codes: 0 = OK, otherwise milo::ErrorCode (errors.hpp:9-20) + 1.
 */
#ifndef MILO_ORACLE_H
#define MILO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OR_OK = 0,
  OR_FORMAT = 1, OR_DATA, OR_IO, OR_SHAPE, OR_RANK, OR_NUMERIC, OR_STAT, OR_PLAN, OR_RANGE,
  OR_CONFIG
};

/* half.hpp:47-158 */
uint16_t or_float_to_half(float f);
float or_half_to_float(uint16_t h);
uint16_t or_double_to_half(double d);
uint16_t or_half_add(uint16_t a, uint16_t b);
uint16_t or_half_sub(uint16_t a, uint16_t b);
uint16_t or_half_mul(uint16_t a, uint16_t b);
uint16_t or_half_fma(uint16_t a, uint16_t b, uint16_t c);

/* pack.cpp:33-68 */
int or_pack32(const uint8_t* codes, size_t n, uint32_t* out3);
void or_unpack32(const uint32_t* w3, uint8_t* out32);
/* pack.cpp:133-139 */
uint64_t or_tiled_position(uint64_t rows, uint64_t cols, uint64_t i, uint64_t j);
/* pack.cpp:97-131,141-178: linear/tiled packing of logical codes, optional
 * plane split; zeros == NULL selects symmetric mode.  Scales/zeros are
 * rounded to binary16 (pack.cpp:89-93). */
int or_pack_matrix(uint64_t rows, uint64_t cols, const uint8_t* codes, const float* scales,
                   const float* zeros, uint64_t group_size, int tiled, int split,
                   uint32_t* words, uint32_t* plane_a, uint32_t* plane_b, uint16_t* scales_h,
                   uint16_t* zeros_h);
/* pack.cpp:196-211 */
int or_unpack_codes(uint64_t rows, uint64_t cols, int layout, int split, const uint32_t* words,
                    const uint32_t* plane_a, const uint32_t* plane_b, uint8_t* out);
/* pack.cpp:224-242 */
void or_fast_dequant_pair(uint32_t word, int pair, int mode, uint16_t* out2);
uint16_t or_symmetric_step(uint16_t s);
uint16_t or_asymmetric_offset(uint16_t s, uint16_t z);
/* pack.cpp:244-295 (mode: 0 symmetric, 1 asymmetric) */
int or_dequant_packed_half(uint64_t rows, uint64_t cols, int layout, int split,
                           uint64_t group_size, const uint32_t* words, const uint32_t* plane_a,
                           const uint32_t* plane_b, const uint16_t* scales,
                           const uint16_t* zeros, int mode, uint16_t* out);

/* quant.cpp:23-76: min/max init + round-half-away quantize, bits=3, g=group */
int or_quantize_minmax(uint64_t rows, uint64_t cols, uint64_t group_size, const float* w,
                       uint8_t* codes, float* scales, float* zeros);

/* lowrank.cpp:89-134 */
int or_symm_int3_quantize(const float* values, uint64_t rows, uint64_t cols,
                          uint64_t group_size, uint8_t* codes, float* scales);
void or_symm_int3_dequantize(uint64_t rows, uint64_t cols, uint64_t group_size,
                             const uint8_t* codes, const float* scales, float* out);

/* The hot path: gemm.cpp:117-199.  Argument structs mirror PackedInt3Matrix
 * (pack.hpp:45-66), Compensator (lowrank.hpp:31-50), GemmConfig (gemm.hpp:17-25). */
typedef struct {
  uint64_t rows, cols;
  int layout; /* 0 linear, 1 tiled16x64 */
  int split;
  int mode; /* 0 symmetric, 1 asymmetric */
  uint64_t group_size;
  const uint32_t* words;
  const uint32_t* plane_a;
  const uint32_t* plane_b;
  const uint16_t* scales;
  const uint16_t* zeros; /* NULL == empty */
} or_packed;

typedef struct {
  uint64_t rows, cols, rank;
  int storage; /* 0 real, 1 symm-int3 */
  const float* U;
  const float* V;
  const uint8_t* qu_codes;
  const float* qu_scales;
  const uint8_t* qvt_codes;
  const float* qvt_scales;
  uint64_t group_size;
} or_comp;

typedef struct {
  int tile_k, tile_n;
  uint64_t group_size;
  int mode;
  int pipeline_depth;
  int materialize_compensator;
} or_gemm_cfg;

int or_gemm_validate(const or_gemm_cfg* cfg);                       /* gemm.cpp:23-30 */
int or_pipeline_tail_check(uint64_t k, const or_gemm_cfg* cfg, int* stages, int max_stages,
                           int* n_stages);                           /* gemm.cpp:32-47 */
int or_gemm_w3a16(const float* A, uint64_t m, uint64_t a_cols, const or_packed* W,
                  const or_comp* comp /* nullable */, const or_gemm_cfg* cfg, float* C);

/* tensor_store.cpp:247-266 */
uint64_t or_matrix_memory_bytes(uint64_t rows, uint64_t cols, uint64_t rank, int bits,
                                uint64_t group_size, int comp_bits);

/* ---- MoE layer (NEW: no reference counterpart) ----
 * Router: top-k by descending fp32 logit, ties to the lower expert id.
 *   score_mode 0 (Mixtral): weights = softmax over the selected top-k logits.
 *   score_mode 1 (DeepSeek): weights = softmax over all E logits, taken at the
 *                            top-k ids, not renormalized.
 * Softmax: w_i = exp(l_i - max) / sum_j exp(l_j - max), fp32, sum ascending. */
/* The MoE gate, logits = half(x) W_gate^T (m x E), in the device's exact
 * fp32 order: per (t, e), 32 lane sums over k = l (mod 32) ascending, then the
 * xor tree 16, 8, 4, 2, 1 (paper_2504_02658_b200/csrc/moe.cuh
 * router_gemm_kernel).  gate: E x d binary16 bits. */
void or_router_gemm(const float* x, uint64_t m, uint64_t d, const uint16_t* gate, int E, float* logits);
void or_router_topk(const float* logits, uint64_t m, int E, int K, int score_mode,
                    int32_t* topk_ids, float* topk_w);

/* Expert FFN: h = silu(x W1 + (x U1) V1) * (x W3 + (x U3) V3); y = h W2 + (h U2) V2,
 * each product through or_gemm_w3a16 (so x and h are rounded to binary16 on
 * entry, gemm.cpp:144-146); silu(a) = a / (1 + expf(-a)) in fp32.
 * out[t] = sum_k topk_w[t,k] * y_{topk_ids[t,k]}[t] accumulated in k order,
 * then + sum_s shared_s(x)[t] (weight 1, shared order).  Rows of expert e are
 * its tokens in ascending token order.  n_threads > 1 runs experts in
 * parallel (results are identical). */
typedef struct {
  or_packed w[3];  /* w1 (d x f), w3 (d x f), w2 (f x d) */
  or_comp c[3];
  int has_comp[3];
} or_expert;

int or_moe_forward(const or_expert* experts, int n_experts, const or_expert* shared,
                   int n_shared, const float* x, uint64_t m, uint64_t d, int K,
                   const int32_t* topk_ids, const float* topk_w, int n_threads, float* out);

#ifdef __cplusplus
}
#endif
#endif
