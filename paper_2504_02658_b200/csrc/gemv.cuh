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
// A warp range is cut into segments at slab boundaries.  Each segment's fp32
// partial (64 x m_pad per matrix) goes to ws[warp][0] (first segment),
// ws[warp][1] (last segment) or full[slab] (a middle segment, which is always a
// whole slab).  gemv_epilogue_kernel then sums each slab's contributors in
// warp order (deterministic: depends only on T and GW), adds t V, and stores.
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
  int32_t gw;                 // total warps of the GEMM grid (grid * GemvCfg::kWarps)
  int32_t pdl_trigger_early;  // let the next grid (e.g. the t = A U kernel) co-run
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
  if (args.pdl_trigger_early) pdl_launch_dependents();

  const int64_t T = pre_u[P];
  const int64_t G = min((int64_t)args.gw, T);
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + warp;
  if (gw >= G) return;
  const int64_t start = range_start(gw, T, G), end = range_start(gw + 1, T, G);

  // ---- per-warp TMA pipeline (lane 0 is the producer of its own warp) ----
  int pp = 0;
  while (pre_u[pp + 1] <= start) ++pp;
  int64_t ppos = start;
  auto issue = [&](int slot) {
    while (pre_u[pp + 1] <= ppos) ++pp;
    const GemvProblem& pr = args.problems[pp];
    const int kts = pr.k / kTileK;
    const int64_t rel = ppos - pre_u[pp];
    const int64_t s = rel / kts, kt = rel - s * kts;
    uint8_t* dst = ring + slot * CF::kSlotBytes;
    mbar_arrive_expect_tx(&bars[slot], CF::kSlotBytes);
#pragma unroll
    for (int mat = 0; mat < NMAT; ++mat)
      bulk_g2s(dst + mat * kTileBytes, pr.w[mat] + (s * kts + kt) * kTileBytes, kTileBytes,
               &bars[slot]);
    bulk_g2s(dst + CF::kSlotW, pr.act + kt * (kMPad * 64), kMPad * 64, &bars[slot]);
    ++ppos;
  };
  if (lane == 0)
    for (int s = 0; s < kSlots && ppos < end; ++s) issue(s);

  const int g = lane >> 2, q = lane & 3;
  int p = 0;
  while (pre_u[p + 1] <= start) ++p;
  int slot = 0;
  uint32_t phase = 0;
  int64_t pos = start;
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

    for (; pos < seg_end; ++pos) {
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
      __syncwarp();
      if (lane == 0 && ppos < end) {
        fence_proxy_async();  // generic reads of this slot before the async overwrite
        issue(slot);
      }
      if (++slot == kSlots) { slot = 0; phase ^= 1; }
    }

    // ---- segment partial -> ws / full ([mat][n 64][m_pad]) ----
    float* dst = partial_ptr(args.ws, args.full, gw, T, G, sb, se, pre_s[p] + (int)s,
                             CF::kPartFloats);
#pragma unroll
    for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float* d0 = dst + (mat * 64 + 16 * i + g) * kMPad + 8 * nt + 2 * q;
          *reinterpret_cast<float2*>(d0) = make_float2(acc[mat][i][nt][0], acc[mat][i][nt][1]);
          *reinterpret_cast<float2*>(d0 + 8 * kMPad) =
              make_float2(acc[mat][i][nt][2], acc[mat][i][nt][3]);
        }
  }
  if (!args.pdl_trigger_early) pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// Fix-up / epilogue: one CTA (256 threads) per slab.  Sums contributors in
// warp order, adds the compensator term t V (v_real, lowrank.cpp:24-32), then
// stores rows (f32/f16) or SwiGLU -> binary16 act tiles of the next GEMM.
// ---------------------------------------------------------------------------
template <int NT, int NMAT>
__global__ void __launch_bounds__(256) gemv_epilogue_kernel(GemvArgs args) {
  using CF = GemvCfg<NT, NMAT>;
  constexpr int kMPad = CF::kMPad;
  __shared__ int32_t pre_u[kMaxProblems + 1];
  __shared__ int32_t pre_s[kMaxProblems + 1];
  __shared__ float vals[NMAT][64][kMPad + 1];
  pdl_wait();
  const int P = min(*args.n_problems, kMaxProblems);
  if (threadIdx.x < 32) problem_prefix(args.problems, P, pre_u, pre_s, threadIdx.x);
  __syncthreads();
  const int slab_id = blockIdx.x;
  if (slab_id >= pre_s[P]) return;
  int lo = 0, hi = P - 1;  // problem of this slab (binary search over pre_s)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre_s[mid] <= slab_id) lo = mid; else hi = mid - 1;
  }
  const int p = lo;
  const GemvProblem& pr = args.problems[p];
  const int kts = pr.k / kTileK;
  const int s = slab_id - pre_s[p];
  const int64_t T = pre_u[P];
  const int64_t G = min((int64_t)args.gw, T);
  const int64_t sb = (int64_t)pre_u[p] + (int64_t)s * kts, se = sb + kts;
  const int64_t w0 = owner_of(sb, T, G), w1 = owner_of(se - 1, T, G);
  constexpr int kMaxContrib = 512;
  __shared__ const float* contrib[kMaxContrib];
  const int nc = (int)(w1 - w0 + 1 < kMaxContrib ? w1 - w0 + 1 : kMaxContrib);  // <= kts
  for (int c = threadIdx.x; c < nc; c += blockDim.x)
    contrib[c] = partial_ptr(args.ws, args.full, w0 + c, T, G, sb, se, slab_id, CF::kPartFloats);
  __syncthreads();
  for (int v = threadIdx.x; v < CF::kPartFloats; v += blockDim.x) {
    float sum = 0.0f;
    for (int c = 0; c < nc; ++c) sum += contrib[c][v];  // warp order: deterministic
    const int mat = v / (64 * kMPad), rem = v % (64 * kMPad);
    vals[mat][rem / kMPad][rem % kMPad] = sum;
  }
  __syncthreads();
  const int n0 = s * kTileN;
  // compensator: vals[:, col] += t (rows x rank) . V^T[col, :], rank in chunks
  // of kRC staged in smem (t rows and the de-quantized V^T slab).
  constexpr int kRC = 64;
  __shared__ float s_t[kMPad][kRC];
  __shared__ float s_v[64][kRC + 1];
#pragma unroll
  for (int mat = 0; mat < NMAT; ++mat) {
    const int rank = pr.rank[mat];
    if (rank > 0 && pr.t[mat] != nullptr) {
      const int col = threadIdx.x & 63, rh = threadIdx.x >> 6;  // 4 row groups
      constexpr int kRowsPer = (kMPad + 3) / 4;
      const uint8_t* vc = pr.vcodes[mat];
      const float* vs = pr.vscales[mat];
      const float* vr = pr.vreal[mat];
      const int gpr = pr.vgpr[mat];
      const float* tt = pr.t[mat];
      const int rows = min(pr.m, kMPad);
      float add[kRowsPer];
#pragma unroll
      for (int r = 0; r < kRowsPer; ++r) add[r] = 0.0f;
      for (int jb = 0; jb < rank; jb += kRC) {
        const int jn = min(kRC, rank - jb);
        for (int v = threadIdx.x; v < kMPad * kRC; v += blockDim.x) {
          const int r = v / kRC, j = v % kRC;
          s_t[r][j] = (r < rows && j < jn) ? tt[r * rank + jb + j] : 0.0f;
        }
        for (int v = threadIdx.x; v < 64 * kRC; v += blockDim.x) {
          const int nn = v / kRC, j = v % kRC;
          float vv = 0.0f;
          if (j < jn) {
            const int64_t n = n0 + nn;
            if (vc) {  // v_real (lowrank.cpp:24-32): step = s * (2/7), v = step * (c - 4)
              const float step = vs[n * gpr + ((jb + j) >> 6)] * (2.0f / 7.0f);
              vv = step * ((float)vc[n * rank + jb + j] - 4.0f);
            } else {
              vv = vr[n * rank + jb + j];
            }
          }
          s_v[nn][j] = vv;
        }
        __syncthreads();
#pragma unroll 8
        for (int j = 0; j < jn; ++j) {
          const float vv = s_v[col][j];
#pragma unroll
          for (int r = 0; r < kRowsPer; ++r) add[r] += s_t[min(rh * kRowsPer + r, kMPad - 1)][j] * vv;
        }
        __syncthreads();
      }
#pragma unroll
      for (int r = 0; r < kRowsPer; ++r) {
        const int row = rh * kRowsPer + r;
        if (row < rows) vals[mat][col][row] += add[r];
      }
    }
  }
  __syncthreads();
  if (pr.kind == kStoreRows) {
    for (int v = threadIdx.x; v < kMPad * 64; v += blockDim.x) {
      const int row = v >> 6, col = v & 63;
      if (row >= pr.m) continue;
      const int orow = pr.row_map ? pr.row_map[row] : row;
      const float val = vals[0][col][row];
      const int64_t off = (int64_t)orow * pr.ldo + n0 + col;
      if (pr.out_dtype == 0)
        reinterpret_cast<float*>(pr.out)[off] = val;
      else
        reinterpret_cast<__half*>(pr.out)[off] = __float2half_rn(val);
    }
  } else {
    uint32_t* outw = reinterpret_cast<uint32_t*>(pr.out);
    for (int v = threadIdx.x; v < kMPad * 32; v += blockDim.x) {
      const int row = v >> 5, cp = (v & 31) * 2;
      uint32_t packed = 0;
      if (row < pr.m) {
        const float h0 = silu_f(vals[0][cp][row]) * vals[NMAT - 1][cp][row];
        const float h1 = silu_f(vals[0][cp + 1][row]) * vals[NMAT - 1][cp + 1][row];
        packed = h2_as_u32(__floats2half2_rn(h0, h1));
      }
      outw[act_word(kMPad, row, n0 + cp)] = packed;
    }
  }
  pdl_launch_dependents();
}

}  // namespace milo_dev
