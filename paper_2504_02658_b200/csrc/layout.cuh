// Device layouts of the B200 INT3 path and the bit-exact register dequant.
//
// ---------------------------------------------------------------------------
// Weight layout ("macro tiles")
// ---------------------------------------------------------------------------
// A weight W is k x n (rows = k = reduction, cols = n = output; the reference's
// orientation, gemm.hpp:43-46).  It is cut into macro tiles of 64 n x 32 k.
// Tiles are stored slab-major: tile (slab S = n/64, kt = k/32) lives at byte
// (S * (k/32) + kt) * 896, so one slab's k-stream is contiguous.
//
// One macro tile = 2048 weights = 896 bytes = 0.4375 B/weight, exactly the
// reference's accounting (3/8 B of codes + 4 B of binary16 scale+zero per
// 64-group, tensor_store.cpp:247-266):
//   [  0, 512)  plane A : per lane 4 x u32 = {u0.w0, u0.w1, u1.w0, u1.w1}
//   [512, 768)  plane B : per lane 2 x u32 = {u0.w2, u1.w2}
//   [768, 896)  meta    : per q (=lane&3) 32 B = for j in {0,1}, h in {0,1}:
//                         {s[k], s[k+1]} {off[k], off[k+1]} (binary16x2),
//                         k = 16j + 8h + 2q
// (the reference's plane split, pack.cpp:163-178, kept as a 2:1 word split).
//
// The tile is "fragment-native" for mma.m16n8k16 with W^T as the A operand
// (rows = n, cols = k): lane l (g = l>>2, q = l&3) owns 32 k-pairs
// p = 16j + 4i + r (j = k-subtile, i = 16-n subtile, r = A register):
//   n = 16i + g + 8(r&1),   k = 16j + 2q + 8(r>>1) + {0: lo, 1: hi}
// Pairs 16j..16j+15 form unit u=j, packed zero-waste into 3 words:
//   pair pp < 15 : word pp/5, slot t = pp%5: lo code bits [3t,3t+3),
//                  hi code bits [16+3t, 16+3t+3)
//   pair pp = 15 : bit b of the lo (hi) code is bit 15 (31) of word b
//
// Per-(k, 64-n group) scale data is pre-folded on the device at repack time:
//   asymmetric: s = scale, off = -round16(s*z)      (pack.cpp:240-242)
//   symmetric : s = round16(scale*2/7), off = -0.0   (pack.cpp:236-238)
// so every weight is w = fma16(c - bias, s, off), bias = 0 (asym) / 4 (sym):
// one correctly rounded binary16 FMA == half_fma / half_mul of the reference
// (gemm.cpp:70-84), i.e. bit-identical de-quantized weights.
//
// ---------------------------------------------------------------------------
// Activation layout ("act tiles")
// ---------------------------------------------------------------------------
// A block of m_pad token rows x k is stored as [k/32][m_pad][32] binary16,
// row = 64 B = 16 words, word w stored at w ^ (4 * ((row >> 1) & 3)) so the
// B-fragment loads of mma.m16n8k16 are bank-conflict free.  One macro tile's
// activations (32 k x m_pad rows) are a contiguous m_pad*64-byte run.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "ptx.cuh"

namespace milo_dev {

constexpr int kTileN = 64;
constexpr int kTileK = 32;
constexpr int kTileBytes = 896;
constexpr int kPlaneAOff = 0;
constexpr int kPlaneBOff = 512;
constexpr int kMetaOff = 768;

// (n, k) offsets inside a macro tile of pair p, lane l, half lh (0 lo, 1 hi).
__host__ __device__ __forceinline__ int pair_n(int lane, int p) {
  const int i = (p >> 2) & 3, r = p & 3, g = lane >> 2;
  return 16 * i + g + 8 * (r & 1);
}
__host__ __device__ __forceinline__ int pair_k(int lane, int p, int lh) {
  const int j = p >> 4, r = p & 3, q = lane & 3;
  return 16 * j + 2 * q + 8 * (r >> 1) + lh;
}
// byte offset of meta half (s or off) for tile-local k
__host__ __device__ __forceinline__ int meta_byte(int kk, bool is_off) {
  const int j = kk >> 4, rem = kk & 15, h = rem >> 3, q = (rem & 7) >> 1, lh = rem & 1;
  return kMetaOff + q * 32 + j * 16 + h * 8 + (is_off ? 4 : 0) + lh * 2;
}

// Activation-tile word address (in u32 units) of (row, k) for m_pad rows.
__host__ __device__ __forceinline__ uint32_t act_word(int m_pad, int row, int k) {
  const int kt = k >> 5, w = (k & 31) >> 1;
  return (uint32_t)kt * (uint32_t)(m_pad * 16) + (uint32_t)row * 16u +
         (uint32_t)(w ^ (4 * ((row >> 1) & 3)));
}

// Normalization constants: lane value after the LOP3 is 1024 + 2^(3t) c.
struct DqConsts {
  __half2 c0;  // -(1024 + bias)
  __half2 c1;  // -(128 + bias), applied after * 1/8
  __half2 c2;  // -(16 + bias),  applied after * 1/64
  __half2 r8;  // 1/8
  __half2 r64; // 1/64
};
__device__ __forceinline__ DqConsts make_dq_consts(int mode) {
  const float bias = mode == 0 ? 4.0f : 0.0f;
  DqConsts c;
  c.c0 = __float2half2_rn(-(1024.0f + bias));
  c.c1 = __float2half2_rn(-(128.0f + bias));
  c.c2 = __float2half2_rn(-(16.0f + bias));
  c.r8 = __float2half2_rn(0.125f);
  c.r64 = __float2half2_rn(1.0f / 64.0f);
  return c;
}

// Exact integer codes (c - bias) of the 16 pairs of one unit, as half2.
// Per pair: one LOP3 ((w & mask) | 0x64006400 -> 1024 + 2^(3t) c in each
// lane) and one HADD2/HFMA2 back to c - bias; slots 3,4 share one shift.
__device__ __forceinline__ void unit_codes(uint32_t W0, uint32_t W1, uint32_t W2,
                                           const DqConsts& k, __half2 (&e)[16]) {
  uint32_t magic = 0x64006400u;
  asm volatile("" : "+r"(magic));  // keep the OR operand in a register (one LOP3 per pair)
  const uint32_t W[3] = {W0, W1, W2};
#pragma unroll
  for (int w = 0; w < 3; ++w) {
    const uint32_t y = W[w] >> 9;
    e[5 * w + 0] = __hadd2(u32_as_h2(and_or<0x00070007u>(W[w], magic)), k.c0);
    e[5 * w + 1] = __hfma2(u32_as_h2(and_or<0x00380038u>(W[w], magic)), k.r8, k.c1);
    e[5 * w + 2] = __hfma2(u32_as_h2(and_or<0x01C001C0u>(W[w], magic)), k.r64, k.c2);
    e[5 * w + 3] = __hadd2(u32_as_h2(and_or<0x00070007u>(y, magic)), k.c0);
    e[5 * w + 4] = __hfma2(u32_as_h2(and_or<0x00380038u>(y, magic)), k.r8, k.c1);
  }
  // virtual pair: bit b of each code is bit 15 (lo) / 31 (hi) of word b
  const uint32_t v = and_or<0x00040004u>(W2 >> 13,
                                         and_or<0x00020002u>(W1 >> 14,
                                                             and_or<0x00010001u>(W0 >> 15, magic)));
  e[15] = __hadd2(u32_as_h2(v), k.c0);
}

// De-quantized weights (binary16 pairs) of one unit: pair pp = 4i + r uses
// the scale pair of h = r >> 1 (S[h], O[h]).
__device__ __forceinline__ void unit_dequant(uint32_t W0, uint32_t W1, uint32_t W2,
                                             const uint32_t (&S)[2], const uint32_t (&O)[2],
                                             const DqConsts& k, uint32_t (&out)[16]) {
  __half2 e[16];
  unit_codes(W0, W1, W2, k, e);
#pragma unroll
  for (int pp = 0; pp < 16; ++pp) {
    const int h = (pp & 3) >> 1;
    out[pp] = h2_as_u32(__hfma2(e[pp], u32_as_h2(S[h]), u32_as_h2(O[h])));
  }
}

// Code (c - bias) of slot t (0..4) of one packed word, as in unit_codes.
template <int T>
__device__ __forceinline__ __half2 slot_code(uint32_t W, uint32_t magic, const DqConsts& k) {
  if (T == 0) return __hadd2(u32_as_h2(and_or<0x00070007u>(W, magic)), k.c0);
  if (T == 1) return __hfma2(u32_as_h2(and_or<0x00380038u>(W, magic)), k.r8, k.c1);
  if (T == 2) return __hfma2(u32_as_h2(and_or<0x01C001C0u>(W, magic)), k.r64, k.c2);
  if (T == 3) return __hadd2(u32_as_h2(and_or<0x00070007u>(W >> 9, magic)), k.c0);
  return __hfma2(u32_as_h2(and_or<0x00380038u>(W >> 9, magic)), k.r8, k.c1);
}

// Half a unit: the 8 pairs pp = 8 IH .. 8 IH + 7 (n subtiles i = 2 IH, 2 IH + 1),
// out[4 il + r] = pair 8 IH + 4 il + r -- for consumers whose threads own only
// half of a unit's 64 n (the prefill kernel's TMEM lane quarters).  Same
// arithmetic per pair as unit_dequant (bit-identical weights).
template <int IH>
__device__ __forceinline__ void half_unit_dequant(uint32_t W0, uint32_t W1, uint32_t W2,
                                                  const uint32_t (&S)[2], const uint32_t (&O)[2],
                                                  const DqConsts& k, uint32_t (&out)[8]) {
  uint32_t magic = 0x64006400u;
  asm volatile("" : "+r"(magic));
  __half2 e[8];
  if (IH == 0) {
    e[0] = slot_code<0>(W0, magic, k);
    e[1] = slot_code<1>(W0, magic, k);
    e[2] = slot_code<2>(W0, magic, k);
    e[3] = slot_code<3>(W0, magic, k);
    e[4] = slot_code<4>(W0, magic, k);
    e[5] = slot_code<0>(W1, magic, k);
    e[6] = slot_code<1>(W1, magic, k);
    e[7] = slot_code<2>(W1, magic, k);
  } else {
    e[0] = slot_code<3>(W1, magic, k);
    e[1] = slot_code<4>(W1, magic, k);
    e[2] = slot_code<0>(W2, magic, k);
    e[3] = slot_code<1>(W2, magic, k);
    e[4] = slot_code<2>(W2, magic, k);
    e[5] = slot_code<3>(W2, magic, k);
    e[6] = slot_code<4>(W2, magic, k);
    const uint32_t v = and_or<0x00040004u>(W2 >> 13,
                                           and_or<0x00020002u>(W1 >> 14,
                                                               and_or<0x00010001u>(W0 >> 15, magic)));
    e[7] = __hadd2(u32_as_h2(v), k.c0);
  }
#pragma unroll
  for (int pp = 0; pp < 8; ++pp) {
    const int h = (pp & 3) >> 1;
    out[pp] = h2_as_u32(__hfma2(e[pp], u32_as_h2(S[h]), u32_as_h2(O[h])));
  }
}

// Raw integer codes of the 16 pairs of one unit (lo in bits 0..7, hi in 8..15).
__device__ __forceinline__ void unit_raw_codes(uint32_t W0, uint32_t W1, uint32_t W2,
                                               uint32_t (&c)[16]) {
  const uint32_t W[3] = {W0, W1, W2};
#pragma unroll
  for (int w = 0; w < 3; ++w)
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const uint32_t lo = (W[w] >> (3 * t)) & 7u, hi = (W[w] >> (16 + 3 * t)) & 7u;
      c[5 * w + t] = lo | (hi << 8);
    }
  const uint32_t lo = ((W0 >> 15) & 1u) | ((W1 >> 14) & 2u) | ((W2 >> 13) & 4u);
  const uint32_t hi = ((W0 >> 31) & 1u) | ((W1 >> 30) & 2u) | ((W2 >> 29) & 4u);
  c[15] = lo | (hi << 8);
}

}  // namespace milo_dev
