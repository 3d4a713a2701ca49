// Support kernels: one-time repack from the reference's packed formats into
// the macro-tile layout, device unpack / de-quantization (bit-exact checks of
// the repack), activation preparation, and the compensator product t = A U.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "gemv.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace milo_dev {

// ---------------------------------------------------------------------------
// Reference stream access: logical (k, n) -> code, for layout linear/tiled16x64
// and split/unsplit words (pack.hpp:62-65, pack.cpp:56-68,133-139).
// ---------------------------------------------------------------------------
struct RefStream {
  const uint32_t* words;
  const uint32_t* plane_a;
  const uint32_t* plane_b;
  uint64_t rows, cols;
  int32_t layout;
  int32_t split;
};

__device__ __forceinline__ uint32_t ref_word(const RefStream& s, uint64_t g, int j) {
  if (!s.split) return s.words[g * 3 + j];
  return j < 2 ? s.plane_a[g * 2 + j] : s.plane_b[g];
}

__device__ __forceinline__ uint32_t ref_code(const RefStream& s, uint64_t k, uint64_t n) {
  uint64_t pos;
  if (s.layout == 0) {
    pos = k * s.cols + n;
  } else {
    const uint64_t tpr = s.cols / 64, ti = k / 16, tj = n / 64, r = k % 16, cc = n % 64;
    pos = (ti * tpr + tj) * 1024 + r * 64 + cc;
  }
  const uint64_t g = pos >> 5;
  const int idx = (int)(pos & 31);
  if (idx < 24) return (ref_word(s, g, idx >> 3) >> (3 * (idx & 7))) & 7u;
  const uint32_t rest = (ref_word(s, g, 0) >> 24) | ((ref_word(s, g, 1) >> 24) << 8) |
                        ((ref_word(s, g, 2) >> 24) << 16);
  return (rest >> (3 * (idx - 24))) & 7u;
}

// One thread per (macro tile, lane): gathers 64 codes, writes 24 B of planes.
__global__ void repack_codes_kernel(RefStream src, uint8_t* dst, uint64_t k, uint64_t n) {
  const uint64_t kts = k / kTileK;
  const uint64_t tiles = (n / kTileN) * kts;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= tiles * 32) return;
  const uint64_t tile = gid >> 5;
  const int lane = (int)(gid & 31);
  const uint64_t slab = tile / kts, kt = tile % kts;
  uint32_t words[2][3] = {{0, 0, 0}, {0, 0, 0}};
  for (int p = 0; p < 32; ++p) {
    const int u = p >> 4, pp = p & 15;
    const uint64_t nn = slab * kTileN + pair_n(lane, p);
    const uint32_t lo = ref_code(src, kt * kTileK + pair_k(lane, p, 0), nn);
    const uint32_t hi = ref_code(src, kt * kTileK + pair_k(lane, p, 1), nn);
    if (pp < 15) {
      const int w = pp / 5, t = pp % 5;
      words[u][w] |= (lo << (3 * t)) | (hi << (16 + 3 * t));
    } else {
      for (int b = 0; b < 3; ++b)
        words[u][b] |= (((lo >> b) & 1u) << 15) | (((hi >> b) & 1u) << 31);
    }
  }
  uint8_t* t = dst + tile * kTileBytes;
  uint32_t* pa = reinterpret_cast<uint32_t*>(t + kPlaneAOff + lane * 16);
  uint32_t* pb = reinterpret_cast<uint32_t*>(t + kPlaneBOff + lane * 8);
  pa[0] = words[0][0];
  pa[1] = words[0][1];
  pa[2] = words[1][0];
  pa[3] = words[1][1];
  pb[0] = words[0][2];
  pb[1] = words[1][2];
}

// One thread per (k row, slab): pre-folded binary16 (s, off) of the group.
//   asym: off = -round16(s * z)                     (pack.cpp:240-242)
//   sym : s' = double_to_half(double(s) * 2 / 7)    (pack.cpp:236-238), off = -0
__global__ void repack_meta_kernel(const uint16_t* scales, const uint16_t* zeros, int mode,
                                   uint8_t* dst, uint64_t k, uint64_t n) {
  const uint64_t slabs = n / kTileN, kts = k / kTileK;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= k * slabs) return;
  const uint64_t row = gid / slabs, slab = gid % slabs;
  const uint64_t qg = row * slabs + slab;  // (row*n + slab*64)/64, gemm.cpp:97
  __half s = __ushort_as_half(scales[qg]);
  __half off;
  if (mode == 1) {
    off = __hneg(__hmul(s, __ushort_as_half(zeros[qg])));
  } else {
    s = __double2half((double)__half2float(s) * 2.0 / 7.0);
    off = __ushort_as_half((unsigned short)0x8000u);
  }
  uint8_t* t = dst + (slab * kts + row / kTileK) * kTileBytes;
  const int kk = (int)(row % kTileK);
  *reinterpret_cast<__half*>(t + meta_byte(kk, false)) = s;
  *reinterpret_cast<__half*>(t + meta_byte(kk, true)) = off;
}

// Device unpack (what=0 -> u8 codes) or de-quantization (what=1 -> binary16)
// of a macro-tile matrix into logical row-major order.  The de-quantization
// runs the exact register path of the GEMM (unit_dequant).
__global__ void unpack_tiles_kernel(const uint8_t* tiles, uint64_t k, uint64_t n, int mode,
                                    int what, void* out) {
  const uint64_t kts = k / kTileK;
  const uint64_t n_tiles = (n / kTileN) * kts;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n_tiles * 32) return;
  const uint64_t tile = gid >> 5;
  const int lane = (int)(gid & 31), q = lane & 3;
  const uint64_t slab = tile / kts, kt = tile % kts;
  const uint8_t* t = tiles + tile * kTileBytes;
  const uint4 pa = *reinterpret_cast<const uint4*>(t + kPlaneAOff + lane * 16);
  const uint2 pb = *reinterpret_cast<const uint2*>(t + kPlaneBOff + lane * 8);
  const DqConsts dq = make_dq_consts(mode);
  for (int j = 0; j < 2; ++j) {
    const uint32_t W0 = j ? pa.z : pa.x, W1 = j ? pa.w : pa.y, W2 = j ? pb.y : pb.x;
    uint32_t vals[16];
    if (what == 0) {
      unit_raw_codes(W0, W1, W2, vals);
    } else {
      const uint4 mm = *reinterpret_cast<const uint4*>(t + kMetaOff + q * 32 + 16 * j);
      const uint32_t S[2] = {mm.x, mm.z}, O[2] = {mm.y, mm.w};
      unit_dequant(W0, W1, W2, S, O, dq, vals);
    }
    for (int pp = 0; pp < 16; ++pp) {
      const int p = 16 * j + pp;
      const uint64_t nn = slab * kTileN + pair_n(lane, p);
      for (int lh = 0; lh < 2; ++lh) {
        const uint64_t kk = kt * kTileK + pair_k(lane, p, lh);
        if (what == 0)
          reinterpret_cast<uint8_t*>(out)[kk * n + nn] = (uint8_t)((vals[pp] >> (8 * lh)) & 0xFFu);
        else
          reinterpret_cast<uint16_t*>(out)[kk * n + nn] = (uint16_t)(vals[pp] >> (16 * lh));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Single-linear preparation: A (m x k, f32/f16) -> binary16 act tiles in
// blocks of m_pad rows (zero padded, gemm.cpp:49-60,144-146), the problem
// table, and zeroed fix-up counters.  One launch; graph-capturable.
// ---------------------------------------------------------------------------
struct LinearPrep {
  const void* A;
  int64_t m, k, lda;
  int32_t a_dtype;
  int32_t m_pad;
  int32_t n_blocks;
  uint32_t* act;           // n_blocks x (k/32) x m_pad x 16 words
  GemvProblem tmpl;        // problem template (block 0); act/t/out/m per block derived
  int64_t act_block_words;
  int64_t t_block_floats;  // per matrix
  int64_t out_block_elems;
  GemvProblem* problems;
  int32_t* n_problems;
  int32_t* counters;
  int32_t n_counters;
  int32_t* t_counters;
  int32_t n_t_counters;
};

__global__ void prep_linear_kernel(LinearPrep a) {
  const int64_t kw = a.k / 2;  // words per row
  const int64_t total = (int64_t)a.n_blocks * a.m_pad * kw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / kw, w = i % kw;
    const int64_t blk = row / a.m_pad;
    const int r = (int)(row % a.m_pad);
    const int64_t kk = 2 * w;
    __half2 v = __floats2half2_rn(0.0f, 0.0f);
    if (row < a.m) {
      if (a.a_dtype == 0) {
        const float* src = reinterpret_cast<const float*>(a.A) + row * a.lda + kk;
        v = __floats2half2_rn(src[0], src[1]);
      } else {
        const __half* src = reinterpret_cast<const __half*>(a.A) + row * a.lda + kk;
        v = __halves2half2(src[0], src[1]);
      }
    }
    a.act[blk * a.act_block_words + act_word(a.m_pad, r, (int)kk)] = h2_as_u32(v);
  }
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = tid; i < a.n_counters; i += (int64_t)gridDim.x * blockDim.x) a.counters[i] = 0;
  for (int64_t i = tid; i < a.n_t_counters; i += (int64_t)gridDim.x * blockDim.x)
    a.t_counters[i] = 0;
  if (tid < a.n_blocks) {
    GemvProblem p = a.tmpl;
    const int b = (int)tid;
    p.act = reinterpret_cast<const uint8_t*>(a.act + b * a.act_block_words);
    for (int mat = 0; mat < 2; ++mat)
      if (p.t[mat]) p.t[mat] = p.t[mat] + b * a.t_block_floats;
    p.m = (int)min((int64_t)a.m_pad, a.m - (int64_t)b * a.m_pad);
    p.out = p.out_dtype == 0
                ? (void*)(reinterpret_cast<float*>(p.out) + b * a.out_block_elems)
                : (void*)(reinterpret_cast<__half*>(p.out) + b * a.out_block_elems);
    a.problems[b] = p;
  }
  if (tid == 0) *a.n_problems = a.n_blocks;
  pdl_launch_dependents();
}

}  // namespace milo_dev
