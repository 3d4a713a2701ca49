// K2: grouped, stream-K, warp-MMA W3A16 kernel for small token blocks
// (decode regime, m_pad = 8*NT <= 16 rows per problem block), with the
// low-rank compensator term and the SwiGLU / store epilogues fused.
//
// Reference semantics: milo::gemm_w3a16 (proj/src/gemm.cpp:117-199) per
// problem: C = A_f16 * dequant(W) + (A_f16 U) V, fp32 accumulation.
//
// Work decomposition.  Each problem (one weight matrix, or a w1|w3 pair for
// SwiGLU, times one block of <= m_pad token rows) is a grid of "units" =
// (slab S of 64 output columns) x (kt = 32-row k step).  Units of all problems
// are concatenated (problem-major, slab-major, kt ascending) into one range of
// T units and CTA c of G owns [c*T/G, (c+1)*T/G) — perfect balance over the
// 148 SMs whatever the mix of matrix shapes / experts.  A CTA range is cut
// into segments at slab boundaries; only its first and last segment can be
// partial slabs.  Partial slabs go through a deterministic fix-up: each
// contributor writes its partial to ws[cta][slot], the last one (atomic
// counter) sums contributors in CTA order and runs the epilogue, then resets
// the counter.  Summation order depends only on (T, G), never on timing.
//
// CTA = 1 producer warp + 8 consumer warps.  The producer streams a segment in
// stages of up to 8 units with cp.async.bulk (TMA engine) into a 4-deep smem
// ring (weights are slab-contiguous; activations are kt-contiguous act tiles);
// consumer warp w de-quantizes unit w of each stage in registers and issues
// mma.m16n8k16 with W^T as the A operand (the tile is fragment-native).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "layout.cuh"
#include "ptx.cuh"

namespace milo_dev {

constexpr int kMaxProblems = 1024;
constexpr int kConsumerWarps = 8;
constexpr int kUnitsPerStage = kConsumerWarps;
constexpr int kStages = 4;
constexpr int kRedStride = 68;  // floats per reduction row (bank-conflict free)

enum GemvKind : int32_t { kStoreRows = 0, kSwigluAct = 1 };

struct GemvProblem {
  const uint8_t* w[2];        // macro-tile base of matrix 0 / 1 (1: SwiGLU w3)
  const uint8_t* act;         // act tiles of this block (m_pad rows, k)
  const float* t[2];          // LoRC t = A U, [m_pad][rank] fp32, or null
  const uint8_t* vcodes[2];   // qVt codes, n x rank (u8), null -> vreal
  const float* vscales[2];    // qVt scales, n x vgpr (f32)
  const float* vreal[2];      // real-storage V^T, n x rank (f32)
  const uint8_t* ucodes[2];   // qU codes, k x rank (u8), null -> ureal
  const float* uscales[2];    // qU scales, k x vgpr (f32)
  const float* ureal[2];      // real-storage U, k x rank (f32)
  int32_t rank[2];
  int32_t vgpr[2];
  int32_t k, n, m;            // m = valid rows of the block
  int32_t mode;               // 0 symmetric, 1 asymmetric
  int32_t kind;               // GemvKind
  int32_t out_dtype;          // kStoreRows: 0 f32, 1 f16
  int64_t ldo;                // kStoreRows: row pitch (elements)
  void* out;                  // kStoreRows: row-major base; kSwigluAct: act tiles (k' = n)
  const int32_t* row_map;     // kStoreRows: output row of block row r (null = r)
};

struct GemvArgs {
  const GemvProblem* problems;
  const int32_t* n_problems;  // device scalar (problem tables may be built on device)
  float* ws;                  // [G][2][NMAT][m_pad][64]
  int32_t* counters;          // one per slab, zero on entry, restored to zero on exit
  int32_t prefetch_before_wait;  // weights do not depend on the previous grid
};

template <int NT, int NMAT>
struct GemvSmem {
  static constexpr int kMPad = 8 * NT;
  static constexpr int kWBytes = kUnitsPerStage * NMAT * kTileBytes;
  static constexpr int kABytes = kUnitsPerStage * kMPad * 64;
  static constexpr int kStageBytes = kWBytes + kABytes;
  static constexpr int kRedFloats = kConsumerWarps * NMAT * kMPad * kRedStride;
  static constexpr int kBytes =
      kStages * kStageBytes + kRedFloats * 4 + 2 * kMaxProblems * 4 + 2 * kStages * 8 + 64;
};

__device__ __forceinline__ int64_t range_start(int64_t c, int64_t T, int64_t G) {
  return c * T / G;
}
__device__ __forceinline__ int64_t cta_of(int64_t x, int64_t T, int64_t G) {
  return ((x + 1) * G - 1) / T;
}

__device__ __forceinline__ float silu_f(float a) { return a / (1.0f + expf(-a)); }

template <int NT, int NMAT>
__global__ void __launch_bounds__(32 * (1 + kConsumerWarps), 1)
    gemv_w3a16_kernel(GemvArgs args) {
  using SM = GemvSmem<NT, NMAT>;
  constexpr int kMPad = SM::kMPad;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stage_base = smem;
  float* red = reinterpret_cast<float*>(smem + kStages * SM::kStageBytes);
  int32_t* pre_units = reinterpret_cast<int32_t*>(red + SM::kRedFloats);
  int32_t* pre_slabs = pre_units + kMaxProblems;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(pre_slabs + kMaxProblems);
  uint64_t* empty_bar = full_bar + kStages;
  int32_t* flag = reinterpret_cast<int32_t*>(empty_bar + kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x, c = blockIdx.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  // The problem table may be produced by the preceding kernel.
  pdl_wait();
  const int P = min(*args.n_problems, kMaxProblems);
  // Exclusive prefix over problems of units and slabs (one warp, sequential chunks).
  if (warp == 0) {
    int32_t carry_u = 0, carry_s = 0;
    for (int base = 0; base < P; base += 32) {
      const int i = base + lane;
      int32_t u = 0, s = 0;
      if (i < P) {
        const GemvProblem& pr = args.problems[i];
        s = pr.n / kTileN;
        u = s * (pr.k / kTileK);
      }
      int32_t iu = u, is = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t tu = __shfl_up_sync(0xffffffffu, iu, o);
        const int32_t ts = __shfl_up_sync(0xffffffffu, is, o);
        if (lane >= o) { iu += tu; is += ts; }
      }
      if (i < P) {
        pre_units[i] = carry_u + iu - u;
        pre_slabs[i] = carry_s + is - s;
      }
      carry_u += __shfl_sync(0xffffffffu, iu, 31);
      carry_s += __shfl_sync(0xffffffffu, is, 31);
    }
    if (lane == 0) {
      pre_units[P] = carry_u;  // P < kMaxProblems is asserted by the host
      pre_slabs[P] = carry_s;
    }
  }
  __syncthreads();
  const int64_t T = pre_units[P];
  const int64_t start = range_start(c, T, G), end = range_start(c + 1, T, G);

  if (warp == 0) {
    // ===================== producer =====================
    if (lane == 0 && start < end) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      int p = 0;
      while (pre_units[p + 1] <= start) ++p;
      int64_t pos = start;
      while (pos < end) {
        const GemvProblem& pr = args.problems[p];
        const int kts = pr.k / kTileK;
        const int64_t rel = pos - pre_units[p];
        const int64_t s = rel / kts;
        const int64_t seg_end = min(end, (int64_t)pre_units[p] + (s + 1) * kts);
        for (int64_t x = pos; x < seg_end; x += kUnitsPerStage) {
          const int cnt = (int)min((int64_t)kUnitsPerStage, seg_end - x);
          const int64_t kt0 = x - pre_units[p] - s * kts;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = stage_base + stage * SM::kStageBytes;
          mbar_arrive_expect_tx(&full_bar[stage],
                                (uint32_t)(cnt * (NMAT * kTileBytes + kMPad * 64)));
#pragma unroll
          for (int mat = 0; mat < NMAT; ++mat)
            bulk_g2s_hint(st + mat * kUnitsPerStage * kTileBytes,
                          pr.w[mat] + (s * kts + kt0) * kTileBytes, (uint32_t)(cnt * kTileBytes),
                          &full_bar[stage], pol);
          bulk_g2s(st + SM::kWBytes, pr.act + kt0 * kMPad * 64, (uint32_t)(cnt * kMPad * 64),
                   &full_bar[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        pos = seg_end;
        while (p < P && pre_units[p + 1] <= pos) ++p;
      }
    }
    return;  // producer warp does not take part in the epilogue
  }

  // ===================== consumers =====================
  const int cw = warp - 1;
  const int ctid = threadIdx.x - 32;  // 0..255
  const int g = lane >> 2, q = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  int p = 0;
  if (start < end)
    while (pre_units[p + 1] <= start) ++p;
  int64_t pos = start;
  while (pos < end) {
    const GemvProblem& pr = args.problems[p];
    const int kts = pr.k / kTileK;
    const int64_t rel = pos - pre_units[p];
    const int64_t s = rel / kts;
    const int64_t slab_begin = (int64_t)pre_units[p] + s * kts;
    const int64_t seg_end = min(end, slab_begin + kts);
    const DqConsts dq = make_dq_consts(pr.mode);

    float acc[NMAT][4][NT][4];
#pragma unroll
    for (int a = 0; a < NMAT; ++a)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[a][i][nt][e] = 0.0f;

    for (int64_t x = pos; x < seg_end; x += kUnitsPerStage) {
      const int cnt = (int)min((int64_t)kUnitsPerStage, seg_end - x);
      mbar_wait(&full_bar[stage], phase);
      if (cw < cnt) {
        const uint8_t* st = stage_base + stage * SM::kStageBytes;
        const uint32_t* act = reinterpret_cast<const uint32_t*>(st + SM::kWBytes + cw * kMPad * 64);
        uint32_t bf[2][NT][2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int row = 8 * nt + g;
            const int sw = 4 * ((row >> 1) & 3);
            bf[j][nt][0] = act[row * 16 + ((8 * j + q) ^ sw)];
            bf[j][nt][1] = act[row * 16 + ((8 * j + q + 4) ^ sw)];
          }
#pragma unroll
        for (int mat = 0; mat < NMAT; ++mat) {
          const uint8_t* tile = st + mat * kUnitsPerStage * kTileBytes + cw * kTileBytes;
          const uint4 pa = *reinterpret_cast<const uint4*>(tile + kPlaneAOff + lane * 16);
          const uint2 pb = *reinterpret_cast<const uint2*>(tile + kPlaneBOff + lane * 8);
          const uint4 m0 = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32);
          const uint4 m1 = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32 + 16);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint4 mm = j == 0 ? m0 : m1;
            const uint32_t S[2] = {mm.x, mm.z}, O[2] = {mm.y, mm.w};
            uint32_t wv[16];
            unit_dequant(j == 0 ? pa.x : pa.z, j == 0 ? pa.y : pa.w, j == 0 ? pb.x : pb.y, S, O,
                         dq, wv);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int nt = 0; nt < NT; ++nt)
                mma_16816(acc[mat][i][nt], &wv[4 * i], bf[j][nt][0], bf[j][nt][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[stage]);
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }

    // ---- segment epilogue: cross-warp reduction (fixed order) ----
    {
      float* mine = red + cw * (NMAT * kMPad * kRedStride);
#pragma unroll
      for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            float* r0 = mine + (mat * kMPad + 8 * nt + 2 * q) * kRedStride + 16 * i + g;
            r0[0] = acc[mat][i][nt][0];
            r0[kRedStride] = acc[mat][i][nt][1];
            r0[8] = acc[mat][i][nt][2];
            r0[kRedStride + 8] = acc[mat][i][nt][3];
          }
    }
    named_bar_sync(1, 32 * kConsumerWarps);
    constexpr int kVals = NMAT * kMPad * 64;
    for (int v = ctid; v < kVals; v += 32 * kConsumerWarps) {
      const int row = v >> 6, col = v & 63;  // row spans (mat, m_pad)
      float sum = 0.0f;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w)
        sum += red[w * (NMAT * kMPad * kRedStride) + row * kRedStride + col];
      red[row * kRedStride + col] = sum;
    }
    named_bar_sync(1, 32 * kConsumerWarps);

    const bool full_slab = (pos == slab_begin) && (seg_end == slab_begin + kts);
    bool do_epilogue = full_slab;
    if (!full_slab) {
      const int slot = (pos == start) ? 0 : 1;
      float* dst = args.ws + ((c * 2 + slot) * NMAT * kMPad) * 64;
      for (int v = ctid; v < kVals; v += 32 * kConsumerWarps)
        dst[v] = red[(v >> 6) * kRedStride + (v & 63)];
      __threadfence();
      named_bar_sync(1, 32 * kConsumerWarps);
      const int64_t c_first = cta_of(slab_begin, T, G);
      const int64_t c_last = cta_of(slab_begin + kts - 1, T, G);
      const int slab_id = pre_slabs[p] + (int)s;
      if (ctid == 0) {
        // contributors = CTAs with a non-empty range inside [c_first, c_last]
        // (when T < G some CTAs own no unit at all)
        int contributors = 0;
        for (int64_t cc = c_first; cc <= c_last; ++cc)
          contributors += range_start(cc, T, G) < range_start(cc + 1, T, G) ? 1 : 0;
        const int old = atomicAdd(&args.counters[slab_id], 1);
        *flag = (old == contributors - 1) ? 1 : 0;
      }
      named_bar_sync(1, 32 * kConsumerWarps);
      do_epilogue = *flag != 0;
      if (do_epilogue) {
        __threadfence();
        for (int v = ctid; v < kVals; v += 32 * kConsumerWarps) {
          float sum = 0.0f;
          for (int64_t cc = c_first; cc <= c_last; ++cc) {
            const int64_t cs = range_start(cc, T, G);
            if (cs >= range_start(cc + 1, T, G)) continue;  // empty range
            const int sl = (cs >= slab_begin) ? 0 : 1;
            sum += __ldcg(args.ws + ((cc * 2 + sl) * NMAT * kMPad) * 64 + v);
          }
          red[(v >> 6) * kRedStride + (v & 63)] = sum;
        }
        if (ctid == 0) args.counters[slab_id] = 0;
        named_bar_sync(1, 32 * kConsumerWarps);
      }
    }

    if (do_epilogue) {
      // ---- compensator: C[:, slab] += t V[:, slab] (v_real, lowrank.cpp:24-32) ----
      const int n0 = (int)s * kTileN;
#pragma unroll
      for (int mat = 0; mat < NMAT; ++mat) {
        const int rank = pr.rank[mat];
        if (rank > 0 && pr.t[mat] != nullptr) {
          // thread -> (column, half of the rows)
          const int col = ctid & 63, rh = ctid >> 6;  // rh 0..3
          const int n = n0 + col;
          const uint8_t* vc = pr.vcodes[mat] ? pr.vcodes[mat] + (int64_t)n * rank : nullptr;
          const float* vs = pr.vcodes[mat] ? pr.vscales[mat] + (int64_t)n * pr.vgpr[mat] : nullptr;
          const float* vr = pr.vcodes[mat] ? nullptr : pr.vreal[mat] + (int64_t)n * rank;
          constexpr int kRowsPer = (kMPad + 3) / 4;
          float add[kRowsPer];
#pragma unroll
          for (int r = 0; r < kRowsPer; ++r) add[r] = 0.0f;
          const float* tt = pr.t[mat];
          for (int jr = 0; jr < rank; ++jr) {
            float vv;
            if (vc) {
              const float step = vs[jr >> 6] * (2.0f / 7.0f);
              vv = step * ((float)vc[jr] - 4.0f);
            } else {
              vv = vr[jr];
            }
#pragma unroll
            for (int r = 0; r < kRowsPer; ++r) {
              const int row = rh * kRowsPer + r;
              if (row < kMPad) add[r] += tt[row * rank + jr] * vv;
            }
          }
#pragma unroll
          for (int r = 0; r < kRowsPer; ++r) {
            const int row = rh * kRowsPer + r;
            if (row < kMPad) red[(mat * kMPad + row) * kRedStride + col] += add[r];
          }
        }
      }
      named_bar_sync(1, 32 * kConsumerWarps);
      // ---- output ----
      if (pr.kind == kStoreRows) {
        for (int v = ctid; v < kMPad * 64; v += 32 * kConsumerWarps) {
          const int row = v >> 6, col = v & 63;
          if (row >= pr.m) continue;
          const int orow = pr.row_map ? pr.row_map[row] : row;
          const float val = red[row * kRedStride + col];
          const int64_t off = (int64_t)orow * pr.ldo + n0 + col;
          if (pr.out_dtype == 0)
            reinterpret_cast<float*>(pr.out)[off] = val;
          else
            reinterpret_cast<__half*>(pr.out)[off] = __float2half_rn(val);
        }
      } else {
        // SwiGLU: h = silu(c1) * c3 -> binary16 act tiles of the next GEMM (k' = n)
        uint32_t* outw = reinterpret_cast<uint32_t*>(pr.out);
        for (int v = ctid; v < kMPad * 32; v += 32 * kConsumerWarps) {
          const int row = v >> 5, cp = (v & 31) * 2;
          uint32_t packed = 0;
          if (row < pr.m) {
            const float h0 = silu_f(red[row * kRedStride + cp]) *
                             red[((NMAT - 1) * kMPad + row) * kRedStride + cp];
            const float h1 = silu_f(red[row * kRedStride + cp + 1]) *
                             red[((NMAT - 1) * kMPad + row) * kRedStride + cp + 1];
            packed = h2_as_u32(__floats2half2_rn(h0, h1));
          }
          outw[act_word(kMPad, row, n0 + cp)] = packed;
        }
      }
    }
    named_bar_sync(1, 32 * kConsumerWarps);  // red is reused by the next segment
    pos = seg_end;
    while (p < P && pre_units[p + 1] <= pos) ++p;
  }
  pdl_launch_dependents();
}

}  // namespace milo_dev
