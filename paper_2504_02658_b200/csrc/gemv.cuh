// K2: grouped, warp-level stream-K, warp-MMA W3A16 kernel for small token
// blocks (decode regime, m_pad = 8*NT <= 16 rows per problem block), plus the
// deterministic fix-up/epilogue kernel that adds the low-rank compensator term
// and applies the SwiGLU / store epilogue.
//
// Reference semantics: milo::gemm_w3a16 (proj/src/gemm.cpp:117-199) per
// problem: C = A_f16 * dequant(W) + (A_f16 U) V, fp32 accumulation.
//
// Work decomposition.  Each problem (one weight matrix, or a w1|w3 pair for
// SwiGLU, times one block of <= m_pad token rows) is a grid of "units" =
// (slab S of 64 output columns) x (kt = 32-row k step).  Units of all problems
// are concatenated (problem-major, slab-major, kt ascending) into one range of
// T units and warp w of the GW = grid*warps-per-CTA warps owns [w*T/GW, (w+1)*T/GW):
// perfect balance over the 148 SMs whatever the mix of shapes / experts.
//
// Each warp runs its own TMA pipeline: lane 0 keeps kSlots cp.async.bulk
// copies (weights 896 B/tile, activations m_pad*64 B) in flight into a private
// smem ring guarded by per-slot mbarriers, so no warp ever waits for another.
// The warp de-quantizes a macro tile in registers (bit-exact binary16 FMA, see
// layout.cuh) and issues mma.m16n8k16 with W^T as the A operand.
//
// A warp range is cut into segments at slab boundaries.  A segment covering a
// whole slab is finished in registers.  Otherwise its fp32 partial (64 x m_pad
// per matrix) goes to ws[warp][0] (first segment of the warp) or ws[warp][1]
// (last segment) and the warp bumps the slab's counter; the last contributor
// re-reads all partials, sums them in warp order (deterministic: depends only
// on T and GW, never on timing), resets the counter and runs the epilogue:
// + t V (LoRC, t = A U from lorc_t_kernel, which completes before this grid
// starts), then SwiGLU -> binary16 act tiles of the next GEMM, or row stores.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "layout.cuh"
#include "ptx.cuh"

namespace milo_dev {

constexpr int kMaxProblems = 1024;

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
  float* ws;                  // [GW][2][NMAT][64][m_pad] segment partials
  float* full;                // [slabs][NMAT][64][m_pad] whole-slab partials
  int32_t* counters;          // one per slab, zero on entry, restored to zero
  int32_t gw;                 // total warps of the GEMM grid (grid * GemvCfg::kWarps)
};

template <int NT, int NMAT>
struct GemvCfg {
  // 16 warps (512 threads, <= 128 registers) unless the accumulators of the
  // 16-row SwiGLU variant need more registers: then 12 warps.
  static constexpr int kWarps = (NT * NMAT >= 4) ? 12 : 16;
  static constexpr int kMPad = 8 * NT;
  static constexpr int kSlots = (NT == 1 && NMAT == 1) ? 6 : 4;
  static constexpr int kSlotW = NMAT * kTileBytes;
  static constexpr int kSlotBytes = kSlotW + kMPad * 64;
  static constexpr int kWarpBytes = kSlots * kSlotBytes;
  static constexpr int kPartFloats = NMAT * 64 * kMPad;
  static constexpr int kScratchFloats = 64 * (kMPad + 1);  // per-warp epilogue scratch
  static constexpr int kBytes = kWarps * kWarpBytes + kWarps * kSlots * 8 +
                                2 * (kMaxProblems + 1) * 4 + 64;
};

__device__ __forceinline__ int64_t range_start(int64_t w, int64_t T, int64_t G) {
  return w * T / G;
}
__device__ __forceinline__ int64_t owner_of(int64_t x, int64_t T, int64_t G) {
  return ((x + 1) * G - 1) / T;
}

__device__ __forceinline__ float silu_f(float a) { return a / (1.0f + expf(-a)); }

// Exclusive prefix (units, slabs) over the problem table, into smem (one warp).
__device__ __forceinline__ void problem_prefix(const GemvProblem* probs, int P, int32_t* pre_u,
                                               int32_t* pre_s, int lane) {
  int32_t carry_u = 0, carry_s = 0;
  for (int base = 0; base < P; base += 32) {
    const int i = base + lane;
    int32_t u = 0, s = 0;
    if (i < P) {
      s = probs[i].n / kTileN;
      u = s * (probs[i].k / kTileK);
    }
    int32_t iu = u, is = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t tu = __shfl_up_sync(0xffffffffu, iu, o);
      const int32_t ts = __shfl_up_sync(0xffffffffu, is, o);
      if (lane >= o) { iu += tu; is += ts; }
    }
    if (i < P) {
      pre_u[i] = carry_u + iu - u;
      pre_s[i] = carry_s + is - s;
    }
    carry_u += __shfl_sync(0xffffffffu, iu, 31);
    carry_s += __shfl_sync(0xffffffffu, is, 31);
  }
  if (lane == 0) {
    pre_u[P] = carry_u;
    pre_s[P] = carry_s;
  }
}

// Where the partial of warp gw for the slab [sb, se) lives.
__device__ __forceinline__ float* partial_ptr(float* ws, float* full, int64_t gw, int64_t T,
                                              int64_t G, int64_t sb, int64_t se, int slab_id,
                                              int part_floats) {
  const int64_t rs = range_start(gw, T, G), re = range_start(gw + 1, T, G);
  if (rs >= sb) return ws + (gw * 2 + 0) * part_floats;  // first segment of the warp
  if (re <= se) return ws + (gw * 2 + 1) * part_floats;  // last segment of the warp
  return full + (int64_t)slab_id * part_floats;          // middle: a whole slab
}

// Epilogue of one slab on the summed accumulator fragments of a warp.  Lane
// (g, q) holds, per matrix, i in 0..3, nt, e in 0..3:
//   column n = 16 i + g + 8 (e >> 1), row = 8 nt + 2 q + (e & 1).
// 1) compensator: acc += t[row, :] . V^T[n0 + n, :]  (v_real, lowrank.cpp:24-32:
//    step = s * (2/7), v = step * (c - 4), or real f32 V)
// 2) kSwigluAct: h = silu(c1) * c3 -> binary16 act tiles (k' = n) of the next
//    GEMM (pairs along k' formed with a shuffle); kStoreRows: f32/f16 rows.
template <int NT, int NMAT>
__device__ __forceinline__ void slab_epilogue(float (&acc)[NMAT][4][NT][4], const GemvProblem& pr,
                                              int n0, int g, int q, int lane, float* scratch) {
  constexpr int kMPad = 8 * NT;
  const int rows = min(pr.m, kMPad);
#pragma unroll
  for (int mat = 0; mat < NMAT; ++mat) {
    const int rank = pr.rank[mat];
    const float* tt = pr.t[mat];
    if (rank <= 0 || tt == nullptr) continue;
    // Lane -> columns (2 lane, 2 lane + 1), every valid row: m x 2 x rank MACs
    // per lane (no work on padding rows), through a per-warp smem scratch
    // [64][m_pad] back into the MMA fragment layout.
    const uint8_t* vc = pr.vcodes[mat];
    const float* vs = pr.vscales[mat];
    const float* vr = pr.vreal[mat];
    const int gpr = pr.vgpr[mat];
    const int64_t nA = n0 + 2 * lane, nB = nA + 1;
    float cA[kMPad], cB[kMPad];
#pragma unroll
    for (int r = 0; r < kMPad; ++r) cA[r] = cB[r] = 0.0f;
    int j = 0;
    if (vc && (rank & 7) == 0) {
      for (; j < rank; j += 8) {  // 8 rank columns per step, one 8-byte code load per column
        const uint2 wa = __ldg(reinterpret_cast<const uint2*>(vc + nA * rank + j));
        const uint2 wb = __ldg(reinterpret_cast<const uint2*>(vc + nB * rank + j));
        const float sa = __ldg(vs + nA * gpr + (j >> 6)) * (2.0f / 7.0f);
        const float sb = __ldg(vs + nB * gpr + (j >> 6)) * (2.0f / 7.0f);
        float va[8], vb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // (float)c - 4 exactly via the 2^23 magic
          const uint32_t ca = ((u < 4 ? wa.x : wa.y) >> (8 * (u & 3))) & 0xFFu;
          const uint32_t cb = ((u < 4 ? wb.x : wb.y) >> (8 * (u & 3))) & 0xFFu;
          va[u] = sa * (__int_as_float(0x4B000000 | ca) - 8388612.0f);
          vb[u] = sb * (__int_as_float(0x4B000000 | cb) - 8388612.0f);
        }
#pragma unroll
        for (int r = 0; r < kMPad; ++r) {
          if (r < rows) {
            const float4 t0 = *reinterpret_cast<const float4*>(tt + r * rank + j);
            const float4 t1 = *reinterpret_cast<const float4*>(tt + r * rank + j + 4);
            const float tv[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              cA[r] += tv[u] * va[u];
              cB[r] += tv[u] * vb[u];
            }
          }
        }
      }
    }
    for (; j < rank; ++j) {
      float va, vb;
      if (vc) {
        va = vs[nA * gpr + (j >> 6)] * (2.0f / 7.0f) * ((float)vc[nA * rank + j] - 4.0f);
        vb = vs[nB * gpr + (j >> 6)] * (2.0f / 7.0f) * ((float)vc[nB * rank + j] - 4.0f);
      } else {
        va = vr[nA * rank + j];
        vb = vr[nB * rank + j];
      }
#pragma unroll
      for (int r = 0; r < kMPad; ++r)
        if (r < rows) {
          cA[r] += tt[r * rank + j] * va;
          cB[r] += tt[r * rank + j] * vb;
        }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kMPad; ++r) {
      scratch[(2 * lane) * (kMPad + 1) + r] = cA[r];
      scratch[(2 * lane + 1) * (kMPad + 1) + r] = cB[r];
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int n = 16 * i + g + 8 * (e >> 1), row = 8 * nt + 2 * q + (e & 1);
          acc[mat][i][nt][e] += scratch[n * (kMPad + 1) + row];
        }
  }
  if (pr.kind == kStoreRows) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = 8 * nt + 2 * q + (e & 1);
          if (row >= pr.m) continue;
          const int orow = pr.row_map ? pr.row_map[row] : row;
          const int64_t off = (int64_t)orow * pr.ldo + n0 + 16 * i + g + 8 * (e >> 1);
          if (pr.out_dtype == 0)
            reinterpret_cast<float*>(pr.out)[off] = acc[0][i][nt][e];
          else
            reinterpret_cast<__half*>(pr.out)[off] = __float2half_rn(acc[0][i][nt][e]);
        }
  } else {
    uint32_t* outw = reinterpret_cast<uint32_t*>(pr.out);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = 8 * nt + 2 * q + (e & 1);
          const float a = acc[0][i][nt][e];
          float h = silu_f(a) * acc[NMAT - 1][i][nt][e];
          if (row >= pr.m) h = 0.0f;
          const float h_next = __shfl_down_sync(0xffffffffu, h, 4);  // column n + 1 (g + 1)
          if ((g & 1) == 0) {
            const int n = n0 + 16 * i + g + 8 * (e >> 1);
            outw[act_word(kMPad, row, n)] = h2_as_u32(__floats2half2_rn(h, h_next));
          }
        }
  }
}

template <int NT, int NMAT>
__global__ void __launch_bounds__(32 * GemvCfg<NT, NMAT>::kWarps, 1)
    gemv_w3a16_kernel(GemvArgs args) {
  using CF = GemvCfg<NT, NMAT>;
  constexpr int kWarpsPerCta = CF::kWarps;
  constexpr int kMPad = CF::kMPad, kSlots = CF::kSlots;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * CF::kWarpBytes;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem + kWarpsPerCta * CF::kWarpBytes) + warp * kSlots;
  int32_t* pre_u = reinterpret_cast<int32_t*>(smem + kWarpsPerCta * CF::kWarpBytes +
                                              kWarpsPerCta * kSlots * 8);
  int32_t* pre_s = pre_u + kMaxProblems + 1;

  if (lane == 0)
    for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
  fence_barrier_init();
  pdl_wait();  // problem table / activations come from the preceding grid
  const int P = min(*args.n_problems, kMaxProblems);
  if (warp == 0) problem_prefix(args.problems, P, pre_u, pre_s, lane);
  __syncthreads();

  const int64_t T = pre_u[P];
  const int64_t G = min((int64_t)args.gw, T);
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + warp;
  if (gw >= G) return;
  const int64_t start = range_start(gw, T, G), end = range_start(gw + 1, T, G);
  int p0 = 0;
  while (pre_u[p0 + 1] <= start) ++p0;

  // ---- per-warp TMA pipeline: lane 0 is the producer of its own warp ----
  // Producer cursor advanced incrementally (no divisions, one problem-struct
  // load per problem change): tile pointers are slab-contiguous along k.
  int pp = p0, p_kt = 0, p_kts = 1;
  const uint8_t* p_w[NMAT];
  const uint8_t* p_act = nullptr;
  const uint8_t* p_act0 = nullptr;
  int32_t p_left = (int32_t)(end - start);
  auto load_problem = [&](int prob, int64_t rel) {
    const GemvProblem& pr = args.problems[prob];
    p_kts = pr.k / kTileK;
    const int64_t s = rel / p_kts;
    p_kt = (int)(rel - s * p_kts);
#pragma unroll
    for (int mat = 0; mat < NMAT; ++mat) p_w[mat] = pr.w[mat] + rel * kTileBytes;
    p_act0 = pr.act;
    p_act = pr.act + p_kt * (kMPad * 64);
  };
  auto issue = [&](int slot) {
    uint8_t* dst = ring + slot * CF::kSlotBytes;
    mbar_arrive_expect_tx(&bars[slot], CF::kSlotBytes);
#pragma unroll
    for (int mat = 0; mat < NMAT; ++mat) {
      bulk_g2s(dst + mat * kTileBytes, p_w[mat], kTileBytes, &bars[slot]);
      p_w[mat] += kTileBytes;
    }
    bulk_g2s(dst + CF::kSlotW, p_act, kMPad * 64, &bars[slot]);
    p_act += kMPad * 64;
    if (--p_left > 0 && ++p_kt == p_kts) {
      p_kt = 0;
      p_act = p_act0;
      if (p_w[0] == args.problems[pp].w[0] + (int64_t)(pre_u[pp + 1] - pre_u[pp]) * kTileBytes) {
        ++pp;  // next problem (skip empty ones)
        while (pre_u[pp + 1] == pre_u[pp]) ++pp;
        load_problem(pp, 0);
      }
    }
  };
  if (lane == 0) {
    load_problem(p0, start - pre_u[p0]);
    for (int s = 0; s < kSlots && p_left > 0; ++s) issue(s);
  }

  const int g = lane >> 2, q = lane & 3;
  int slot = 0;
  uint32_t phase = 0;
  int64_t pos = start;
  int p = p0;
  while (pos < end) {
    while (pre_u[p + 1] <= pos) ++p;
    const GemvProblem& pr = args.problems[p];
    const int kts = pr.k / kTileK;
    const int64_t s = (pos - pre_u[p]) / kts;
    const int64_t sb = (int64_t)pre_u[p] + s * kts, se = sb + kts;
    const int64_t seg_end = min(end, se);
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

    for (int32_t left = (int32_t)(seg_end - pos); left > 0; --left) {
      mbar_wait(&bars[slot], phase);
      const uint8_t* st = ring + slot * CF::kSlotBytes;
      const uint32_t* act = reinterpret_cast<const uint32_t*>(st + CF::kSlotW);
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
        const uint8_t* tile = st + mat * kTileBytes;
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
      // Every LDS of this slot has been consumed by the MMAs above, so the slot
      // can be refilled once all lanes are past this point.
      __syncwarp();
      if (lane == 0 && p_left > 0) issue(slot);
      if (++slot == kSlots) { slot = 0; phase ^= 1; }
    }
    pos = seg_end;

    // ---- segment partial -> ws / full ([mat][n 64][m_pad], fragment order) ----
    // Plain stores: the fix-up kernel that reads them is the next grid.
    float* dst = partial_ptr(args.ws, args.full, gw, T, G, sb, se, pre_s[p] + (int)s,
                             CF::kPartFloats);
#pragma unroll
    for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float* d0 = dst + (mat * 64 + 16 * i + g) * kMPad + 8 * nt + 2 * q;
          __stcg(reinterpret_cast<float2*>(d0), make_float2(acc[mat][i][nt][0], acc[mat][i][nt][1]));
          __stcg(reinterpret_cast<float2*>(d0 + 8 * kMPad),
                 make_float2(acc[mat][i][nt][2], acc[mat][i][nt][3]));
        }
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// Fix-up + epilogue: one WARP per slab (8 per CTA).  Sums the slab's
// contributor partials in warp order (deterministic), then slab_epilogue
// (+ t V, SwiGLU / store).  Every contributor's loads for a slab are issued
// before any is consumed.
// ---------------------------------------------------------------------------
constexpr int kEpiWarps = 8;

template <int NT, int NMAT>
__global__ void __launch_bounds__(32 * kEpiWarps) gemv_epilogue_kernel(GemvArgs args) {
  using CF = GemvCfg<NT, NMAT>;
  constexpr int kMPad = CF::kMPad;
  __shared__ int32_t pre_u[kMaxProblems + 1];
  __shared__ int32_t pre_s[kMaxProblems + 1];
  __shared__ float scratch_all[kEpiWarps][CF::kScratchFloats];
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = min(*args.n_problems, kMaxProblems);
  if (warp == 0) problem_prefix(args.problems, P, pre_u, pre_s, lane);
  __syncthreads();
  const int slab_id = blockIdx.x * kEpiWarps + warp;
  if (slab_id >= pre_s[P]) return;
  int lo = 0, hi = P - 1;  // problem of this slab (binary search over pre_s)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre_s[mid] <= slab_id) lo = mid; else hi = mid - 1;
  }
  const GemvProblem& pr = args.problems[lo];
  const int kts = pr.k / kTileK;
  const int s = slab_id - pre_s[lo];
  const int64_t T = pre_u[P];
  const int64_t G = min((int64_t)args.gw, T);
  const int64_t sb = (int64_t)pre_u[lo] + (int64_t)s * kts, se = sb + kts;
  const int64_t w0 = owner_of(sb, T, G), w1 = owner_of(se - 1, T, G);
  const int g = lane >> 2, q = lane & 3;
  // Contributor pointers first (lane c computes contributor w0 + c), then all
  // lanes load every contributor's fragment values: for each chunk of up to
  // 8 contributors the loads are issued before the in-order adds.
  const int nc = (int)(w1 - w0 + 1);
  float acc[NMAT][4][NT][4];
#pragma unroll
  for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[mat][i][nt][e] = 0.0f;
  for (int c0 = 0; c0 < nc; c0 += 32) {
    const float* myp = nullptr;
    if (c0 + lane < nc)
      myp = partial_ptr(args.ws, args.full, w0 + c0 + lane, T, G, sb, se, slab_id, CF::kPartFloats);
    const int cn = min(32, nc - c0);
    constexpr int kU = (NT * NMAT >= 4) ? 1 : (NT * NMAT == 2 ? 2 : 4);  // loads in flight
    for (int cb = 0; cb < cn; cb += kU) {
      float2 v[kU][NMAT][4][NT][2];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const float* src = reinterpret_cast<const float*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(myp), min(cb + u, cn - 1)));
#pragma unroll
        for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const float* s0 = src + (mat * 64 + 16 * i + g) * kMPad + 8 * nt + 2 * q;
              if (cb + u < cn) {
                v[u][mat][i][nt][0] = __ldcg(reinterpret_cast<const float2*>(s0));
                v[u][mat][i][nt][1] = __ldcg(reinterpret_cast<const float2*>(s0 + 8 * kMPad));
              } else {
                v[u][mat][i][nt][0] = v[u][mat][i][nt][1] = make_float2(0.0f, 0.0f);
              }
            }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              acc[mat][i][nt][0] += v[u][mat][i][nt][0].x;
              acc[mat][i][nt][1] += v[u][mat][i][nt][0].y;
              acc[mat][i][nt][2] += v[u][mat][i][nt][1].x;
              acc[mat][i][nt][3] += v[u][mat][i][nt][1].y;
            }
    }
  }
  slab_epilogue<NT, NMAT>(acc, pr, s * kTileN, g, q, lane, scratch_all[warp]);
  pdl_launch_dependents();
}

}  // namespace milo_dev
