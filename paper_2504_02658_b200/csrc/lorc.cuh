// Compensator product t = A_f16 U for every (problem, matrix) with rank > 0:
// the "U x" half of the LoRC term U.(V.x) (the reference's gemm.cpp:185-192,
// T = Ah . U); the "T V" half is folded into the GEMM epilogue (gemv.cuh).
//
// U is the reference's u_real (lowrank.cpp:19-22): symm-int3 codes (u8, k x r)
// with f32 scales per 64-group along the rank, step = s*(2/7),
// u = step*(c-4), or real f32 U.
//
// Grid = (problem*2 + mat, k-chunk).  Each CTA stages its chunk of U rows, their
// scales and the matching activation tiles with three cp.async.bulk copies (one
// mbarrier), computes the chunk's m_pad x r partial with a fixed-order
// reduction over 8 k-slices, and the last CTA of the item (atomic counter)
// sums the chunk partials in chunk order: deterministic.
//
// Launch order: ... -> lorc_t_kernel -> GEMM (whose epilogues read t).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "gemv.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace milo_dev {

constexpr int kLorcThreads = 256;
constexpr int kLorcSmemU = 32 * 1024;  // bytes of U rows per chunk
constexpr int kLorcMaxRows = 64;       // many small chunks: latency, not throughput, matters

struct LorcArgs {
  const GemvProblem* problems;
  const int32_t* n_problems;
  float* partial;     // [items][chunks_max][m_pad][rank_max]
  int32_t* counters;  // one per item (problem*2 + mat), zero on entry, reset after use
  int32_t m_pad;
  int32_t chunks_max;
  int32_t rank_max;
};

// Rows per chunk for a given rank / element size: a multiple of 32 (one act
// tile), at most kLorcMaxRows, and the U rows fit kLorcSmemU.
__host__ __device__ __forceinline__ int lorc_rows(int rank, int elem_bytes) {
  int rows = kLorcSmemU / (rank * elem_bytes);
  rows = rows > kLorcMaxRows ? kLorcMaxRows : rows;
  rows &= ~31;
  return rows < 32 ? 32 : rows;
}

__global__ void __launch_bounds__(kLorcThreads) lorc_t_kernel(LorcArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float s_red[8][16][33];
  __shared__ uint64_t bar;
  __shared__ int s_last;
  pdl_wait();
  const int item = blockIdx.x, chunk = blockIdx.y;
  const int p = item >> 1, mat = item & 1;
  const int tid = threadIdx.x;
  if (p >= *a.n_problems) return;
  const GemvProblem& pr = a.problems[p];
  const int rank = pr.rank[mat];
  float* tout = const_cast<float*>(pr.t[mat]);
  if (rank <= 0 || tout == nullptr) return;
  const uint8_t* uc = pr.ucodes[mat];
  const int ebytes = uc ? 1 : 4;
  const int rows = lorc_rows(rank, ebytes);
  const int k = pr.k, m_pad = a.m_pad, m = min(pr.m, m_pad);
  const int nch = (k + rows - 1) / rows;
  if (chunk >= nch) return;
  const int k0 = chunk * rows, kc = min(rows, k - k0);
  const int gpr = (rank + 63) / 64;

  // ---- stage U rows, scales and activation tiles (bulk async copies) ----
  uint8_t* s_u = smem;                                         // kc x rank (u8 or f32)
  float* s_sc = reinterpret_cast<float*>(smem + kLorcSmemU);   // kc x gpr
  uint32_t* s_act = reinterpret_cast<uint32_t*>(smem + kLorcSmemU + kLorcMaxRows * 16 * 4);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    const uint32_t ub = (uint32_t)(kc * rank * ebytes);
    const uint32_t sb = uc ? (uint32_t)(kc * gpr * 4) : 0u;
    const uint32_t ab = (uint32_t)(kc / 32) * m_pad * 64;
    mbar_arrive_expect_tx(&bar, ub + sb + ab);
    if (uc) {
      bulk_g2s(s_u, uc + (int64_t)k0 * rank, ub, &bar);
      bulk_g2s(s_sc, pr.uscales[mat] + (int64_t)k0 * gpr, sb, &bar);
    } else {
      bulk_g2s(s_u, pr.ureal[mat] + (int64_t)k0 * rank, ub, &bar);
    }
    bulk_g2s(s_act, pr.act + (int64_t)(k0 / 32) * m_pad * 64, ab, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);

  // ---- chunk partial: thread -> (rank column j of the pass, k slice ks) ----
  float* part = a.partial + ((int64_t)item * a.chunks_max + chunk) * m_pad * a.rank_max;
  const int jj = tid & 31, ks = tid >> 5;
  const int per = ((kc + 15) / 16) * 2;  // even rows per k slice
  const int kb = min(kc, ks * per), ke = min(kc, kb + per);
  for (int jb = 0; jb < rank; jb += 32) {
    const int j = jb + jj;
    float acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = 0.0f;
    if (j < rank) {
      // rows in pairs (one act word = binary16 pair (k, k+1)); kb, ke are even
      for (int kk = kb; kk < ke; kk += 2) {
        float u0, u1;
        if (uc) {
          // (float)c - 4 exactly via the 2^23 magic: float(0x4B000000 | c) = 2^23 + c
          const float st0 = s_sc[kk * gpr + (j >> 6)] * (2.0f / 7.0f);
          const float st1 = s_sc[(kk + 1) * gpr + (j >> 6)] * (2.0f / 7.0f);
          u0 = st0 * (__int_as_float(0x4B000000 | s_u[kk * rank + j]) - 8388612.0f);
          u1 = st1 * (__int_as_float(0x4B000000 | s_u[(kk + 1) * rank + j]) - 8388612.0f);
        } else {
          u0 = reinterpret_cast<const float*>(s_u)[kk * rank + j];
          u1 = reinterpret_cast<const float*>(s_u)[(kk + 1) * rank + j];
        }
        const int kt = kk >> 5, wrd = (kk & 31) >> 1;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (r < m) {
            const uint32_t w = s_act[kt * (m_pad * 16) + r * 16 + (wrd ^ (4 * ((r >> 1) & 3)))];
            const float2 xv = __half22float2(u32_as_h2(w));
            acc[r] += xv.x * u0;
            acc[r] += xv.y * u1;
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) s_red[ks][r][jj] = acc[r];
    __syncthreads();
    for (int v = tid; v < m_pad * 32; v += kLorcThreads) {
      const int r = v >> 5, c = v & 31;
      if (jb + c < rank)
        part[r * a.rank_max + jb + c] =
            ((s_red[0][r][c] + s_red[1][r][c]) + (s_red[2][r][c] + s_red[3][r][c])) +
            ((s_red[4][r][c] + s_red[5][r][c]) + (s_red[6][r][c] + s_red[7][r][c]));
    }
    __syncthreads();
  }

  // ---- last CTA of the item sums the chunk partials in chunk order ----
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&a.counters[item], 1) == nch - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // Sum the nch chunk partials of the m x rank valid values: `groups` thread
  // groups each sum a contiguous run of chunks (8 loads in flight), then the
  // group sums are added in group order (fixed: deterministic).
  const float* base = a.partial + (int64_t)item * a.chunks_max * m_pad * a.rank_max;
  const int64_t stride = (int64_t)m_pad * a.rank_max;
  float* s_grp = &s_red[0][0][0];  // reused: [8][256]
  const int nv = m * rank;
  // depends on rank (not m) so every row's summation order is independent of
  // the batch size: padded and unpadded runs stay bit-identical
  const int groups = max(1, min(8, kLorcThreads / rank));
  const int per_pass = kLorcThreads / groups;
  for (int vb = 0; vb < nv; vb += per_pass) {
    const int vl = tid % per_pass, gi = tid / per_pass, v = vb + vl;
    if (v < nv && gi < groups) {
      const int r = v / rank, j = v % rank;
      const float* src = base + r * a.rank_max + j;
      const int c0 = gi * nch / groups, c1 = (gi + 1) * nch / groups;
      float s = 0.0f;
      int ch = c0;
      for (; ch + 8 <= c1; ch += 8) {
        float x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldcg(src + (ch + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += x[u];
      }
      for (; ch < c1; ++ch) s += __ldcg(src + ch * stride);
      s_grp[gi * 256 + vl] = s;
    }
    __syncthreads();
    if (tid < per_pass && vb + tid < nv) {
      float s = 0.0f;
      for (int gg = 0; gg < groups; ++gg) s += s_grp[gg * 256 + tid];
      const int v = vb + tid;
      tout[(v / rank) * rank + v % rank] = s;
    }
    __syncthreads();
  }
  if (tid == 0) a.counters[item] = 0;
}

constexpr int kLorcDynSmem = kLorcSmemU + kLorcMaxRows * 16 * 4 + (kLorcMaxRows / 32) * 16 * 64;

}  // namespace milo_dev
