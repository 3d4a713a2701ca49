// K2': the decode-regime MoE layer (and single linear) in ONE persistent launch.
//
// Reference semantics, per matrix: milo::gemm_w3a16 (proj/src/gemm.cpp:117-199)
//   C = half(A) * dequant(W) + (half(A) U) V, fp32 accumulation,
// composed into the top-k routed expert layer defined in SURVEY.md section 8b
// (the reference has no MoE layer):
//   h_e = half(silu(x W1_e + t1 V1_e) * (x W3_e + t3 V3_e)),  y_e = h_e W2_e + t2 V2_e,
//   out[t] = sum_k w[t,k] y_{e(t,k)}[t] + sum_shared y_s[t].
//
// Grid = one CTA per SM (cooperative launch: all CTAs co-resident).  A CTA has
// C consumer warps and one producer warp whose lane c feeds consumer c's ring
// of cp.async.bulk slots (full / empty mbarriers per slot).  A call:
//
//  stage 0  every CTA, redundantly: router top-k (or the given routing), the
//           block table (one block per touched expert, tokens ascending;
//           shared experts: all tokens) and the per-phase problem tables.
//  phase 1  warp-level stream-K over the units of
//             [LoRC pseudo-slabs: t = x U, 16 rank columns x 32 k per unit]
//             [w1|w3 slabs: 64 n x 32 k per unit, both matrices per unit]
//           Activations are copied per token row straight from x (binary16).
//           A slab's last-arriving contributor (atomic counter) sums the
//           contributors' partials in warp order (deterministic) and
//           finishes it: pseudo -> t (t-ready flag when all its chunks are
//           in); real -> + t V (tensor cores, fp32-exact split), SwiGLU -> the
//           block's h tiles (block-ready flag when all its slabs are in).
//  phase 2  the same over [t2 = h U2 pseudo-slabs][w2 slabs] -> y rows; the
//           last block finishing a d-slab runs the weighted combine -> out.
// The units of a phase are split evenly over all consumer warps of the grid
// whatever the mix of experts / ranks.  The producer never blocks: it issues
// phase-2 weight copies while phase 1 drains and adds each unit's activation
// copy once that block's h is published.
//
// Waits never form a cycle: consumers finish all pseudo units (which wait for
// nothing) before any real unit, and all of phase 1 (finisher duty included)
// before any phase-2 unit; the producer only polls.  Spin waits are bounded
// and trap instead of hanging.
//
// LoRC on the tensor cores without losing fp32 accuracy: U / V codes are
// exact binary16 integers c - 4; the fp32 side (x * step for t = x U, and t for
// t V) is split into hi + lo binary16 halves, two MMAs, fp32 accumulation.
// Real-storage factors are split hi + lo instead.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "gemv.cuh"
#include "layout.cuh"
#include "moe.cuh"
#include "ptx.cuh"

namespace milo_dev {

#ifndef DEC_SLOTS
#define DEC_SLOTS 2  // ring slots per warp (MoE decode)
#endif

#ifndef DEC_MAX_BLOCKS
#define DEC_MAX_BLOCKS 96
#endif
constexpr int kDecMaxBlocks = DEC_MAX_BLOCKS;  // (expert, 16-token chunk) blocks per launch
constexpr int kDecMaxTok = 16;                    // token rows per block (NT = 2)
constexpr int kDecMaxM = 64;                      // MoE decode path: m <= 64 (experts' tokens split into blocks)
constexpr int kDecMaxEntries = 384;               // m * K routed entries (DeepSeek top-6 at m = 64)
constexpr int kDecKC = 8;                         // max k-tiles (32 k each) per ring slot
#ifndef DEC_SLOT_BYTES
#define DEC_SLOT_BYTES 8192
#endif
constexpr int kDecSlotW = DEC_SLOT_BYTES;         // weight / pseudo-tile bytes per slot
constexpr int kPseudoInt3Bytes = 640;             // 512 B codes + 32 f32 steps
constexpr int kPseudoRealBytes = 2048;            // hi / lo binary16 fragments
constexpr int kVftInt3Bytes = 1024;               // per (slab, 16-rank step)
constexpr int kVftRealBytes = 4096;

// One quantized matrix + compensator in device layout (built at create time).
//   upt  : U pseudo tiles [r16/16][k/32], fragment-native A operand (rows =
//          16 rank columns, cols = 32 k): int3 -> per lane 16 code bytes
//          [ks][reg][2] then 32 f32 steps (s * 2/7 of the 64-group); real ->
//          per lane [ks][hi 4 regs][lo 4 regs].
//   vft  : V^T fragment tiles [n/64][r16/16]: per lane [i 0..3][8 code bytes]
//          (int3) or [i][hi 4][lo 4] (real); rows = n, cols = rank.
//   vstep: [n][gpr] f32 steps of V (int3 only).
struct DecMat {
  const uint8_t* w;
  const uint8_t* upt;
  const uint8_t* vft;
  const float* vstep;
  int32_t k, n, rank, r16, gpr, real, mode, pad;
};

struct DecExpert {
  DecMat m[3];  // w1, w3, w2 (single linear: m[0])
};

// Cross-warp values (stream-K partials, LoRC t) are tagged 64-bit words
// {f32 bits, epoch}: a naturally aligned b64 store is single-copy atomic, so a
// reader that sees the call's epoch in a word sees its value -- no fences, no
// counters; writers never wait.
struct DecWs {
  uint64_t* part;       // [2 phases][G warps][2 segments][part_stride] tagged
  uint64_t* t;          // [blocks][3][m_pad][r16_max] tagged
  __half* h;            // [blocks][m_pad][f_max] row-major (phase-2 activations)
  float* Y;             // [m*K + S*m][d]
  __half* xrep;         // [grid][m][d] CTA-private binary16 copies of x (null: read x directly)
  int32_t* cnt1;        // phase-1 slab counters
  int32_t* cnt2;        // phase-2 slab counters
  int32_t* tcnt;        // [blocks][3]
  int32_t* bcnt;        // [blocks]
  int32_t* ccnt;        // [d/64]
  int32_t* tflag;       // [blocks][3]   (epoch-valued)
  int32_t* bflag;       // [blocks]
  int32_t* hflag;       // [blocks][f_max / 64]  h slab ready (epoch-valued)
  int64_t part_stride;  // floats per (phase, warp, segment)
  int32_t r16_max;
  int32_t f_max;
};

struct DecArgs {
  int32_t moe;                 // 1: MoE layer, 0: single linear
  int32_t m;                   // token rows of this call
  int32_t epoch;
  int32_t gw;                  // consumer warps of the grid
  // MoE
  const float* logits;         // m x E (router) or null (routing given)
  const int32_t* ids_in;       // m x K given routing (-1 = unused slot)
  const float* wts_in;
  int32_t* ids_out;            // optional routing outputs
  float* wts_out;
  int32_t E, K, S, score_mode;
  const DecExpert* experts;    // E routed then S shared (device); linear: null, uses lin
  DecExpert lin;               // the single linear's matrix (m[0])
  // activations / output
  const void* x;               // rows of x (x_dtype) -- binary16 when xrep is null
  int32_t x_dtype;             // 0 f32, 1 f16
  int32_t d;                   // MoE hidden size (linear: k)
  int64_t ldx;
  void* out;
  int32_t out_dtype;
  int64_t ldo;
  DecWs ws;
  long long* dbg;              // optional per-warp timeline (globaltimer ns), [warp][16]
  int32_t dbg_flags;           // experiments: bit 4 no V prefetch, bit 5 no activation loads
};

// Work of a phase = the concatenated k-tiles of its problems' slabs; warp gw
// of Gp owns tiles [gw T / Gp, (gw + 1) T / Gp) (balanced to one tile) and
// streams them in ring slots of <= kc tiles that never cross a slab.
struct DProb {
  const uint8_t* src[2];  // pseudo: U tiles; real: weight tiles of matrix 0 / 1
  int32_t t0, s0;         // exclusive prefix of tiles / slabs within the phase
  int32_t n_slabs;        // 0 = empty entry (rank-0 compensator)
  int16_t kind, mat;      // kind 0 pseudo, 1 real; mat = matrix index 0..2
  int16_t b, kc;          // block; max tiles per ring slot
  int16_t ktiles, tb;     // 32-k tiles per slab; bytes per tile (896 real, 640 / 2048 pseudo)
};

struct DBlock {
  int32_t e;
  int32_t rows;
  int32_t chunk;             // this block = the expert's tokens [chunk * m_pad, ...)
  int16_t xrow[kDecMaxTok];  // x row of each block row (MoE: token; linear: row)
  int16_t slot[kDecMaxTok];  // output row (MoE: Y slot; linear: C row)
};

template <int NT, int NMAT1>
struct DecCfg {
  static constexpr int kMPad = 8 * NT;
#ifdef DEC_CONS12
  static constexpr int kCons = NT == 1 ? 12 : 8;  // warps (each feeds its own ring)
#else
  static constexpr int kCons = (NT == 1 && NMAT1 == 1) ? 12 : 8;  // warps (each feeds its own ring)
#endif
  static constexpr int kWarps = kCons;
  static constexpr int kSlotBytes = kDecSlotW;
  static constexpr int kSlots = kCons == 12 ? 2 : DEC_SLOTS;
  static constexpr int kRing = kCons * kSlots * kSlotBytes;
  static constexpr int kPartMax = 2 * 64 * kMPad;  // floats of the largest partial
  // smem carve-up
  static constexpr int kOffBars = kRing;  // full [kCons][kSlots]
  static constexpr int kOffProbs = kOffBars + kCons * kSlots * 8;
  // (expert, chunk) blocks: the single linear needs <= 16 (its 12-warp ring
  // leaves no room for more tables)
  static constexpr int kMaxBlocks = NMAT1 == 2 ? kDecMaxBlocks : 16;
  static constexpr int kMaxProbs = 3 * kMaxBlocks;  // per phase
  static constexpr int kOffBlocks = kOffProbs + 2 * kMaxProbs * (int)sizeof(DProb);
  static constexpr int kOffRoute = kOffBlocks + kMaxBlocks * (int)sizeof(DBlock);
  static constexpr int kRouteBytes = kDecMaxEntries * 4 * 2 + 256 * 8 + 64;
  static constexpr int kOffMats = kOffRoute + kRouteBytes;  // DecExpert per block (smem copy)
  static constexpr int kMats = kMaxBlocks;
  static constexpr int kBytes = kOffMats + kMats * (int)sizeof(DecExpert);
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// two u8 codes (bytes 0,1 or 2,3 of w) -> half2 (c0 - 4, c1 - 4), exact.
__device__ __forceinline__ uint32_t codes_h2(uint32_t w, bool upper) {
  const uint32_t v = prmt(w, 0x64646464u, upper ? 0x4342u : 0x4140u);  // 1024 + c
  return h2_as_u32(__hadd2(u32_as_h2(v), __float2half2_rn(-1028.0f)));
}
// fp32 pair -> binary16 hi + lo with hi + lo == (a, b) to ~2^-22.
__device__ __forceinline__ void split_h2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 f = __half22float2(h);
  hi = h2_as_u32(h);
  lo = h2_as_u32(__floats2half2_rn(a - f.x, b - f.y));
}

#ifndef DEC_WARM
#define DEC_WARM 1  // finisher code warm-up by the grid's last warp
#endif
#ifndef DEC_W2_PREFETCH
#define DEC_W2_PREFETCH 0  // L2 prefetch of the phase-2 weights during phase 1 (measured slower: 87 -> 92 us)
#endif
#ifndef DEC_FIN_LOW
#define DEC_FIN_LOW 1  // slab finisher: 1 = lowest contributor (its piece ends its range, 2 segments)
#endif
#ifndef DEC_TIMERS
#define DEC_TIMERS 0  // per-warp cycle counters in the debug timeline (tools/dbg_timeline.py)
#endif

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DEC_DBG(i)                                                                     \
  do {                                                                                 \
    if (a.dbg != nullptr && (threadIdx.x & 31) == 0)                                   \
      a.dbg[((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 16 + (i)] = \
          globaltimer();                                                               \
  } while (0)

__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acqrel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Bounded spin until *p == v (relaxed polls, one acquiring load at the end).
// Traps after ~2 s instead of hanging.
__device__ __forceinline__ void spin_until(const int* p, int v) {
  if (ld_relaxed_gpu(p) != v) {
    const long long t0 = clock64();
    while (ld_relaxed_gpu(p) != v) {
      __nanosleep(32);
      if (clock64() - t0 > 4000000000LL) __trap();
    }
  }
  (void)ld_acquire_gpu(p);
}
__device__ __forceinline__ void st_tagged2(uint64_t* p, float a, float b, int epoch) {
  const uint64_t hi = (uint64_t)(uint32_t)epoch << 32;
  asm volatile("st.global.cg.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(hi | __float_as_uint(a)),
               "l"(hi | __float_as_uint(b))
               : "memory");
}
__device__ __forceinline__ void st_tagged1(uint64_t* p, float a, int epoch) {
  asm volatile("st.global.cg.b64 [%0], %1;" ::"l"(p), "l"(((uint64_t)(uint32_t)epoch << 32) | __float_as_uint(a))
               : "memory");
}
// Loads two tagged words; true when both carry `epoch`.
__device__ __forceinline__ bool ld_tagged2(const uint64_t* p, int epoch, float2& v) {
  uint64_t a, b;
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  v = make_float2(__uint_as_float((uint32_t)a), __uint_as_float((uint32_t)b));
  return (uint32_t)(a >> 32) == (uint32_t)epoch && (uint32_t)(b >> 32) == (uint32_t)epoch;
}
__device__ __forceinline__ void warp_backoff(long long t0) {
  __nanosleep(64);
  if (clock64() - t0 > 4000000000LL) __trap();
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Phase 2: wait until the h slabs covering k in [k0, k1) of block b are
// published (lane j polls slab k0 / 64 + j; relaxed polls, the h loads that
// follow go to L2 with ld.cg and are issued only after the flags were seen).
__device__ __forceinline__ void wait_h(const int32_t* hflag, int k0, int k1, int epoch, int lane) {
  const int j0 = k0 >> 6, nj = ((k1 - 1) >> 6) - j0 + 1;
  bool ok = lane >= nj || ld_relaxed_gpu(hflag + j0 + lane) == epoch;
  if (__all_sync(0xffffffffu, ok)) return;
  const long long t0 = clock64();
  while (!__all_sync(0xffffffffu, ok)) {
    __nanosleep(64);
    ok = ok || ld_relaxed_gpu(hflag + j0 + lane) == epoch;
    if (clock64() - t0 > 4000000000LL) __trap();
  }
}

// Same, with the readiness already seen kept in a warp-uniform 32-slab window
// (base, mask): once a segment's flags have been seen, later slots need no
// global round trip.  nflags bounds the block's flag array.
struct HWin {
  int base;
  uint32_t mask;
};
__device__ __forceinline__ void wait_h_cached(const int32_t* hflag, int nflags, HWin& w, int k0, int k1, int epoch,
                                              int lane) {
  const int j0 = k0 >> 6, j1 = (k1 - 1) >> 6;
  if (j0 < w.base || j1 >= w.base + 32) {
    w.base = j0;
    w.mask = 0u;
  }
  const int n = j1 - j0 + 1;
  const uint32_t need = (n >= 32 ? 0xffffffffu : ((1u << n) - 1u)) << (j0 - w.base);
  if ((w.mask & need) == need) return;
  const long long t0 = clock64();
  for (;;) {
    const int j = w.base + lane;
    const bool ok = ((w.mask >> lane) & 1u) || (j < nflags && ld_relaxed_gpu(hflag + j) == epoch);
    w.mask = __ballot_sync(0xffffffffu, ok);
    if ((w.mask & need) == need) return;
    __nanosleep(64);
    if (clock64() - t0 > 4000000000LL) __trap();
  }
}

// Stream-K range arithmetic in 32 bits (tiles per phase x warps < 2^32, checked
// at launch): 64-bit divisions are software routines on the finisher's chain.
__device__ __forceinline__ int rng_at(int w, int T, int G) {
  return (int)(((uint32_t)w * (uint32_t)T) / (uint32_t)G);
}
__device__ __forceinline__ int rng_owner(int x, int T, int G) {
  return (int)((((uint32_t)x + 1u) * (uint32_t)G - 1u) / (uint32_t)T);
}

// B fragments of one 32-k tile, loaded straight from the activation rows
// (binary16, row-major, L1/L2 resident): v[j][nt] = {x[row][k + 16 j + 2q .. +1],
// x[row][k + 16 j + 2q + 8 .. +9]}, row = 8 nt + g.  rowp[nt] == nullptr -> padding
// row (zeros).
template <int NT>
struct BTile {
  uint32_t v[2][NT][2];
};
template <int NT, bool CG = false>
__device__ __forceinline__ void load_btile(BTile<NT>& b, const __half* const (&rowp)[NT], int k, bool on, int q) {
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      uint32_t b0 = 0u, b1 = 0u;
      if (on && rowp[nt] != nullptr) {
        const __half* p = rowp[nt] + k + 16 * j + 2 * q;
        if (CG) {  // written by other SMs during this call: read at L2
          b0 = __ldcg(reinterpret_cast<const unsigned int*>(p));
          b1 = __ldcg(reinterpret_cast<const unsigned int*>(p + 8));
        } else {
          b0 = *reinterpret_cast<const uint32_t*>(p);
          b1 = *reinterpret_cast<const uint32_t*>(p + 8);
        }
      }
      b.v[j][nt][0] = b0;
      b.v[j][nt][1] = b1;
    }
}

// One k-tile of a real unit: NMAT macro tiles (matrix mat's tile at tile + mat * mstride).
template <int NT, int NMAT, int NA, int A0 = 0>
__device__ __forceinline__ void tile_real(const uint8_t* tile0, int mstride, const BTile<NT>& b,
                                          float (&acc)[NA][4][NT][4], const DqConsts& dq, int lane) {
  const int q = lane & 3;
#pragma unroll
  for (int mat = 0; mat < NMAT; ++mat) {
    const uint8_t* tile = tile0 + mat * mstride;
    const uint4 pa = *reinterpret_cast<const uint4*>(tile + kPlaneAOff + lane * 16);
    const uint2 pb = *reinterpret_cast<const uint2*>(tile + kPlaneBOff + lane * 8);
    const uint4 m0 = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32);
    const uint4 m1 = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32 + 16);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint4 mm = j == 0 ? m0 : m1;
      const uint32_t S[2] = {mm.x, mm.z}, O[2] = {mm.y, mm.w};
      uint32_t wv[16];
      unit_dequant(j == 0 ? pa.x : pa.z, j == 0 ? pa.y : pa.w, j == 0 ? pb.x : pb.y, S, O, dq, wv);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mma_16816(acc[A0 + mat][i][nt], &wv[4 * i], b.v[j][nt][0], b.v[j][nt][1]);
    }
  }
}

// One k-tile of a pseudo unit: t chunk (16 rank cols x tokens) += U^T chunk (16 x 32 k) * x.
template <int NT, int NA>
__device__ __forceinline__ void tile_pseudo(const uint8_t* st, bool real, const BTile<NT>& b,
                                            float (&acc)[NA][4][NT][4], int lane) {
  const int q = lane & 3;
  if (!real) {
    const uint4 cw = *reinterpret_cast<const uint4*>(st + lane * 16);
    const float* steps = reinterpret_cast<const float*>(st + 512);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t w0 = j == 0 ? cw.x : cw.z, w1 = j == 0 ? cw.y : cw.w;
      const uint32_t A[4] = {codes_h2(w0, false), codes_h2(w0, true), codes_h2(w1, false), codes_h2(w1, true)};
      const float2 s0 = *reinterpret_cast<const float2*>(steps + 16 * j + 2 * q);
      const float2 s1 = *reinterpret_cast<const float2*>(steps + 16 * j + 2 * q + 8);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float2 x0 = __half22float2(u32_as_h2(b.v[j][nt][0]));
        const float2 x1 = __half22float2(u32_as_h2(b.v[j][nt][1]));
        uint32_t h0, l0, h1, l1;
        split_h2(x0.x * s0.x, x0.y * s0.y, h0, l0);
        split_h2(x1.x * s1.x, x1.y * s1.y, h1, l1);
        mma_16816(acc[0][0][nt], A, h0, h1);
        mma_16816(acc[0][0][nt], A, l0, l1);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint4 hi = *reinterpret_cast<const uint4*>(st + lane * 64 + j * 32);
      const uint4 lo = *reinterpret_cast<const uint4*>(st + lane * 64 + j * 32 + 16);
      const uint32_t AH[4] = {hi.x, hi.y, hi.z, hi.w}, AL[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        mma_16816(acc[0][0][nt], AH, b.v[j][nt][0], b.v[j][nt][1]);
        mma_16816(acc[0][0][nt], AL, b.v[j][nt][0], b.v[j][nt][1]);
      }
    }
  }
}

// acc[i][nt][e] += (t V)^T of the slab's 64 columns:  t = [m_pad][r16max] fp32
// (global), V fragment tiles of the slab.  int3: per 64-rank group g_r,
// D = c'(V) * split(t) on the tensor cores, then acc += step[n][g_r] * D.
// All loads of a group are issued before its MMAs (one round trip per group).
template <int NT>
__device__ __forceinline__ void add_tv(float (&acc)[4][NT][4], const DecMat& M, const uint64_t* t,
                                       int r16max, int slab, int lane, int epoch, bool dry) {
  const int g = lane >> 2, q = lane & 3;
  const int nks = M.r16 >> 4;
  const int n0 = slab * 64;
  const uint8_t* vb = M.vft + (int64_t)slab * nks * (M.real ? kVftRealBytes : kVftInt3Bytes);
  constexpr int kB = 2;  // rank steps whose loads are in flight together
  for (int kb = 0; kb * kB < nks; ++kb) {
    const int gr = (kb * kB) >> 2;  // 64-rank group of this batch
    const int nk = min(kB, nks - kb * kB);
    float D[4][NT][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) D[i][nt][e] = 0.0f;
    float sv[8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        sv[2 * i + h] = M.real ? 1.0f : __ldg(M.vstep + (int64_t)(n0 + 16 * i + g + 8 * h) * M.gpr + gr);
    if (!M.real) {
      float2 tv[kB][NT][2];
      uint4 cv[kB][2];
#pragma unroll
      for (int kk = 0; kk < kB; ++kk) {
        if (kk >= nk) continue;
        const int ks = kb * kB + kk;
        const uint4* src = reinterpret_cast<const uint4*>(vb + (int64_t)ks * kVftInt3Bytes + lane * 32);
        cv[kk][0] = __ldg(src);
        cv[kk][1] = __ldg(src + 1);
      }
      // t (published by the pseudo slabs' finishers): poll the tags
      for (long long t0 = 0;;) {
        bool ok = true;
#pragma unroll
        for (int kk = 0; kk < kB; ++kk) {
          if (kk >= nk) continue;
          const int ks = kb * kB + kk;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const uint64_t* tr = t + (8 * nt + g) * r16max + 16 * ks + 2 * q;
            ok &= ld_tagged2(tr, epoch, tv[kk][nt][0]);
            ok &= ld_tagged2(tr + 8, epoch, tv[kk][nt][1]);
          }
        }
        if (__all_sync(0xffffffffu, ok || dry)) break;
        if (t0 == 0) t0 = clock64();
        warp_backoff(t0);
      }
#pragma unroll
      for (int kk = 0; kk < kB; ++kk) {
        if (kk >= nk) continue;
        uint32_t bh[NT][2], bl[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          split_h2(tv[kk][nt][0].x, tv[kk][nt][0].y, bh[nt][0], bl[nt][0]);
          split_h2(tv[kk][nt][1].x, tv[kk][nt][1].y, bh[nt][1], bl[nt][1]);
        }
        const uint32_t cw[8] = {cv[kk][0].x, cv[kk][0].y, cv[kk][0].z, cv[kk][0].w,
                                cv[kk][1].x, cv[kk][1].y, cv[kk][1].z, cv[kk][1].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t A[4] = {codes_h2(cw[2 * i], false), codes_h2(cw[2 * i], true),
                                 codes_h2(cw[2 * i + 1], false), codes_h2(cw[2 * i + 1], true)};
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma_16816(D[i][nt], A, bh[nt][0], bh[nt][1]);
            mma_16816(D[i][nt], A, bl[nt][0], bl[nt][1]);
          }
        }
      }
    } else {
      for (int kk = 0; kk < nk; ++kk) {
        const int ks = kb * kB + kk;
        uint32_t bh[NT][2], bl[NT][2];
        float2 v0[NT], v1[NT];
        for (long long t0 = 0;;) {
          bool ok = true;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const uint64_t* tr = t + (8 * nt + g) * r16max + 16 * ks + 2 * q;
            ok &= ld_tagged2(tr, epoch, v0[nt]);
            ok &= ld_tagged2(tr + 8, epoch, v1[nt]);
          }
          if (__all_sync(0xffffffffu, ok || dry)) break;
          if (t0 == 0) t0 = clock64();
          warp_backoff(t0);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          split_h2(v0[nt].x, v0[nt].y, bh[nt][0], bl[nt][0]);
          split_h2(v1[nt].x, v1[nt].y, bh[nt][1], bl[nt][1]);
        }
        const uint4* src = reinterpret_cast<const uint4*>(vb + (int64_t)ks * kVftRealBytes + lane * 128);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 hi = __ldg(src + 2 * i), lo = __ldg(src + 2 * i + 1);
          const uint32_t AH[4] = {hi.x, hi.y, hi.z, hi.w}, AL[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma_16816(D[i][nt], AH, bh[nt][0], bh[nt][1]);
            mma_16816(D[i][nt], AH, bl[nt][0], bl[nt][1]);
            mma_16816(D[i][nt], AL, bh[nt][0], bh[nt][1]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[i][nt][2 * h] += sv[2 * i + h] * D[i][nt][2 * h];
          acc[i][nt][2 * h + 1] += sv[2 * i + h] * D[i][nt][2 * h + 1];
        }
  }
}

// ---------------------------------------------------------------- stage 0
// Every CTA, redundantly: routing (or the given routing), the block table and
// the per-phase problem tables in shared memory.  Ends with __syncthreads().
template <int NT, int NMAT1, bool MOE>
__device__ __forceinline__ void dec_stage0(const DecArgs& a) {
  using CF = DecCfg<NT, NMAT1>;
  constexpr int kMPad = CF::kMPad;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  DProb* probs = reinterpret_cast<DProb*>(smem + CF::kOffProbs);
  DBlock* blocks = reinterpret_cast<DBlock*>(smem + CF::kOffBlocks);
  int32_t* r_ids = reinterpret_cast<int32_t*>(smem + CF::kOffRoute);
  float* r_wts = reinterpret_cast<float*>(r_ids + kDecMaxEntries);
  unsigned long long* emask = reinterpret_cast<unsigned long long*>(r_wts + kDecMaxEntries);  // token bits
  int32_t* sc = reinterpret_cast<int32_t*>(emask + 256);
  const DecExpert* experts = MOE ? a.experts : &a.lin;
  const int m = a.m;
  if (MOE) {
    const int K = a.K, E = a.E;
    for (int e = tid; e < 256; e += blockDim.x) emask[e] = 0ull;
    if (a.logits != nullptr) {
      for (int t = warp; t < m; t += blockDim.x >> 5)
        topk_regs(a.logits + (int64_t)t * E, E, K, a.score_mode, r_ids + t * K, r_wts + t * K, lane);
    } else {
      for (int i = tid; i < m * K; i += blockDim.x) {
        r_ids[i] = a.ids_in[i];
        r_wts[i] = a.wts_in[i];
      }
    }
    __syncthreads();
    if (blockIdx.x == 0 && a.logits != nullptr && a.ids_out != nullptr)
      for (int i = tid; i < m * K; i += blockDim.x) {
        a.ids_out[i] = r_ids[i];
        a.wts_out[i] = r_wts[i];
      }
    for (int i = tid; i < m * K; i += blockDim.x) {
      const int e = r_ids[i];
      if (e >= 0 && e < E) atomicOr(&emask[e], 1ull << (i / K));
    }
    __syncthreads();
    if (warp == 0) {  // touched experts ascending (their tokens in chunks of m_pad), then shared experts
      int nb = 0;
      const int nse = E + a.S;
      for (int e0 = 0; e0 < nse; e0 += 32) {
        const int e = e0 + lane;
        const int cnt = e < E ? __popcll(emask[e]) : (e < nse ? m : 0);
        const int nch = (cnt + kMPad - 1) / kMPad;
        int incl = nch;  // inclusive scan of the chunk counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        for (int c = 0; c < nch; ++c) {
          if (nb + incl - nch + c < CF::kMaxBlocks) {
            blocks[nb + incl - nch + c].e = e;
            blocks[nb + incl - nch + c].chunk = c;
          }
        }
        nb += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) sc[0] = min(nb, CF::kMaxBlocks);
    }
    __syncthreads();
    const int nb = sc[0];
    for (int b = tid; b < nb; b += blockDim.x) {
      DBlock& B = blocks[b];
      const int e = B.e;
      const unsigned long long mask = e < E ? emask[e] : (m >= 64 ? ~0ull : ((1ull << m) - 1ull));
      int r = 0, skip = B.chunk * kMPad;
      for (int t = 0; t < m && r < kMPad; ++t) {
        if (!(mask >> t & 1ull)) continue;
        if (skip > 0) {
          --skip;
          continue;
        }
        int slot;
        if (e < E) {
          int kk = 0;
          for (int k = 0; k < K; ++k)
            if (r_ids[t * K + k] == e) kk = k;
          slot = t * K + kk;
        } else {
          slot = m * K + (e - E) * m + t;
        }
        B.xrow[r] = (int16_t)t;
        B.slot[r] = (int16_t)slot;
        ++r;
      }
      B.rows = r;
      for (; r < kDecMaxTok; ++r) B.xrow[r] = B.slot[r] = -1;
    }
  } else {
    const int nb = (m + kMPad - 1) / kMPad;
    if (tid == 0) sc[0] = nb;
    for (int b = tid; b < nb; b += blockDim.x) {
      DBlock& B = blocks[b];
      B.e = 0;
      B.chunk = 0;
      B.rows = min(kMPad, m - b * kMPad);
      for (int r = 0; r < kDecMaxTok; ++r) {
        const bool on = r < B.rows;
        B.xrow[r] = on ? (int16_t)(b * kMPad + r) : (int16_t)-1;
        B.slot[r] = B.xrow[r];
      }
    }
  }
  __syncthreads();
  const int nb = sc[0];
  DecExpert* bx = reinterpret_cast<DecExpert*>(smem + CF::kOffMats);
  for (int i = tid; i < min(nb, CF::kMats) * 3; i += blockDim.x) bx[i / 3].m[i % 3] = experts[blocks[i / 3].e].m[i % 3];
  __syncthreads();
  // problem entries, one thread each: phase 1 [pseudo (b, mat)][real b], phase 2
  // [pseudo b][real b]; rank-0 pseudo entries stay as empty (n_slabs = 0) entries.
  // kc = tiles per ring slot: as many as fit kDecSlotW (both matrices of a w1|w3 slab).
  const int nm1 = MOE ? 2 : 1;
  const int np1 = nb * (nm1 + 1), np2 = MOE ? nb * 2 : 0;
  for (int i = tid; i < np1 + np2; i += blockDim.x) {
    const int ph = i < np1 ? 0 : 1;
    const int j = ph == 0 ? i : i - np1;
    DProb& P = probs[ph * CF::kMaxProbs + j];
    int b, mat, kind;
    if (ph == 0) {
      kind = j < nb * nm1 ? 0 : 1;
      b = kind == 0 ? j / nm1 : j - nb * nm1;
      mat = kind == 0 ? j % nm1 : 0;
    } else {
      kind = j < nb ? 0 : 1;
      b = kind == 0 ? j : j - nb;
      mat = 2;
    }
    const DecExpert& X = bx[b];
    const DecMat& M = X.m[mat];
    P.kind = (int16_t)kind;
    P.mat = (int16_t)mat;
    P.b = (int16_t)b;
    P.ktiles = (int16_t)(M.k / kTileK);
    if (kind == 0) {
      P.n_slabs = M.rank > 0 ? M.r16 / 16 : 0;
      P.src[0] = M.upt;
      P.src[1] = nullptr;
      P.tb = (int16_t)(M.real ? kPseudoRealBytes : kPseudoInt3Bytes);
    } else {
      P.n_slabs = M.n / kTileN;
      P.src[0] = M.w;
      P.src[1] = (MOE && ph == 0) ? X.m[1].w : nullptr;
      P.tb = (int16_t)kTileBytes;
    }
    const int nmu = (kind == 1 && ph == 0 && MOE) ? NMAT1 : 1;
    P.kc = (int16_t)min(kDecKC, kDecSlotW / (P.tb * nmu));
  }
  __syncthreads();
  if (warp < 2) {  // exclusive prefix of units / slabs per phase (warp ph)
    const int ph = warp;
    const int n = ph == 0 ? np1 : np2;
    DProb* PP = probs + ph * CF::kMaxProbs;
    int cu = 0, cs = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const int s = i < n ? PP[i].n_slabs : 0;
      const int u = i < n ? s * PP[i].ktiles : 0;
      int iu = u, is = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tu = __shfl_up_sync(0xffffffffu, iu, o);
        const int ts = __shfl_up_sync(0xffffffffu, is, o);
        if (lane >= o) {
          iu += tu;
          is += ts;
        }
      }
      if (i < n) {
        PP[i].t0 = cu + iu - u;
        PP[i].s0 = cs + is - s;
      }
      cu += __shfl_sync(0xffffffffu, iu, 31);
      cs += __shfl_sync(0xffffffffu, is, 31);
    }
    if (lane == 0) {
      sc[1 + ph] = n;
      sc[3 + ph] = cu;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- segment end
// A warp's segment of slab s of problem p ended with partial accumulators accl
// ([NMAT1][4][NT][4], local memory).  Publishes the partial (or keeps it when the
// warp covered the whole slab); the slab's last contributor sums all partials in
// warp order and finishes the slab.
template <int NT, int NMAT1, bool MOE, int NM>
__device__ __forceinline__ void dec_finish(const DecArgs& a, float* accs, int ph, int p, int s, int start,
                                        int end, int Gp, int Tp, int gw, int G, bool dry) {
  using CF = DecCfg<NT, NMAT1>;
  constexpr int kMPad = CF::kMPad;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  // the segment's accumulators, parked in the warp's just-consumed ring slot
  float acc[NM][4][NT][4];
#pragma unroll
  for (int x = 0; x < NM; ++x)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[x][i][nt][e] = accs[(((x * 4 + i) * NT + nt) * 4 + e) * 32 + lane];
  const DProb& P = reinterpret_cast<const DProb*>(smem + CF::kOffProbs)[ph * CF::kMaxProbs + p];
  const DBlock* blocks = reinterpret_cast<const DBlock*>(smem + CF::kOffBlocks);
  const int32_t* r_ids = reinterpret_cast<const int32_t*>(smem + CF::kOffRoute);
  const float* r_wts = reinterpret_cast<const float*>(r_ids + kDecMaxEntries);
  const int32_t* sc = reinterpret_cast<const int32_t*>(reinterpret_cast<const unsigned long long*>(r_wts + kDecMaxEntries) + 256);
  const DecExpert* experts = MOE ? a.experts : &a.lin;
  const DecWs& W = a.ws;
  const int epoch = a.epoch;
  const int d = a.d;
  const bool pseudo = P.kind == 0;
  const int nmat = pseudo ? 1 : NM;
  const bool fdbg = !dry && ph == 0 && end <= P.t0 + (s + 1) * P.ktiles;  // the warp's last phase-1 segment
#define FIN_DBG(i) \
  if (fdbg) DEC_DBG(i)
  FIN_DBG(8);
  const int ni = pseudo ? 1 : 4;
  const int sb = P.t0 + s * P.ktiles, se = sb + P.ktiles;
  uint64_t* part_base = W.part + (int64_t)ph * G * 2 * W.part_stride;
  if (dry || !(start <= sb && end >= se)) {  // not the sole contributor
    // The slab's finisher is fixed: the lowest contributor (its piece of the
    // slab ends its range and it usually has two segments, so it arrives last;
    // the others' pieces are their whole range or the first segment of theirs,
    // which never wait on anything -- no cycles).  The others publish tagged
    // partials and move on.
    int w0 = rng_owner(sb, Tp, Gp), w1 = rng_owner(se - 1, Tp, Gp);
    const int w1end = rng_at(w1 + 1, Tp, Gp);
    int fin = DEC_FIN_LOW ? w0 : ((w1end <= se || w1 == w0) ? w1 : w1 - 1);
    if (dry) {  // code warm-up: the finisher path with one (pretend-ready) other contributor
      w0 = gw - 1;
      w1 = fin = gw;
    }
    if (gw != fin) {
      uint64_t* dst = part_base + ((int64_t)gw * 2 + (start > sb ? 0 : 1)) * W.part_stride;
#pragma unroll
      for (int mat = 0; mat < NM; ++mat)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (mat >= nmat || i >= ni) continue;
            uint64_t* d0 = dst + (mat * 64 + 16 * i + g) * kMPad + 8 * nt + 2 * q;
            st_tagged2(d0, acc[mat][i][nt][0], acc[mat][i][nt][1], epoch);
            st_tagged2(d0 + 8 * kMPad, acc[mat][i][nt][2], acc[mat][i][nt][3], epoch);
          }
      FIN_DBG(9);
      return;
    }
    FIN_DBG(9);
    // sum all contributors in warp order (deterministic); this warp's own
    // accumulators are re-read from the parked copy in shared memory
#pragma unroll
    for (int mat = 0; mat < NM; ++mat) {
      if (mat >= nmat) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[mat][i][nt][e] = 0.0f;
      for (int w = w0; w <= w1; ++w) {
        if (w == gw) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (i < ni) acc[mat][i][nt][e] += accs[(((mat * 4 + i) * NT + nt) * 4 + e) * 32 + lane];
          continue;
        }
        const int rs = rng_at(w, Tp, Gp);
        const uint64_t* src = part_base + ((int64_t)w * 2 + (rs > sb ? 0 : 1)) * W.part_stride;
        constexpr int kI = NT == 1 ? 4 : 2;  // 16-column groups polled together (registers)
#pragma unroll
        for (int i0 = 0; i0 < 4; i0 += kI) {
          if (i0 >= ni) continue;
          float2 v[kI][NT][2];
          for (long long t0 = 0;;) {
            bool ok = true;
#pragma unroll
            for (int ii = 0; ii < kI; ++ii)
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                if (i0 + ii >= ni) continue;
                const uint64_t* s0 = src + (mat * 64 + 16 * (i0 + ii) + g) * kMPad + 8 * nt + 2 * q;
                ok &= ld_tagged2(s0, epoch, v[ii][nt][0]);
                ok &= ld_tagged2(s0 + 8 * kMPad, epoch, v[ii][nt][1]);
              }
            if (__all_sync(0xffffffffu, ok || dry)) break;
            if (t0 == 0) t0 = clock64();
            warp_backoff(t0);
          }
#pragma unroll
          for (int ii = 0; ii < kI; ++ii)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              if (i0 + ii >= ni) continue;
              acc[mat][i0 + ii][nt][0] += v[ii][nt][0].x;
              acc[mat][i0 + ii][nt][1] += v[ii][nt][0].y;
              acc[mat][i0 + ii][nt][2] += v[ii][nt][1].x;
              acc[mat][i0 + ii][nt][3] += v[ii][nt][1].y;
            }
        }
      }
    }
  }

  FIN_DBG(10);
  const DBlock& B = blocks[P.b];
  const DecExpert& X = reinterpret_cast<const DecExpert*>(smem + CF::kOffMats)[P.b];
  if (pseudo) {
    // t[b][mat][row][16 s + j]: D rows = rank j (g, g + 8), cols = token rows
    uint64_t* tb = W.t + ((int64_t)P.b * 3 + P.mat) * kMPad * W.r16_max;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 16 * s + g + 8 * (e >> 1), row = 8 * nt + 2 * q + (e & 1);
        if (!dry) st_tagged1(tb + row * W.r16_max + j, acc[0][0][nt][e], epoch);
      }
    return;
  }
  // real slab: + t V for each matrix with a compensator (t polled by tag)
  const int nmr = NM;
  FIN_DBG(11);
#pragma unroll
  for (int mat = 0; mat < NM; ++mat) {
    if (mat >= nmr) continue;
    const int mi = ph == 0 ? mat : 2;
    const DecMat& M = X.m[mi];
    if (M.rank <= 0) continue;
    add_tv<NT>(acc[mat], M, W.t + ((int64_t)P.b * 3 + mi) * kMPad * W.r16_max, W.r16_max, s, lane, epoch, dry);
  }
  FIN_DBG(12);
  const int n0 = s * kTileN;
  if (!MOE) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = 8 * nt + 2 * q + (e & 1);
          if (row >= B.rows || dry) continue;
          const int64_t off = (int64_t)B.slot[row] * a.ldo + n0 + 16 * i + g + 8 * (e >> 1);
          if (a.out_dtype == 0)
            reinterpret_cast<float*>(a.out)[off] = acc[0][i][nt][e];
          else
            reinterpret_cast<__half*>(a.out)[off] = __float2half_rn(acc[0][i][nt][e]);
        }
  } else if (ph == 0) {
    // SwiGLU -> h rows of block b (k' = n), padding rows zero
    __half* hb = W.h + (int64_t)P.b * kMPad * W.f_max;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = 8 * nt + 2 * q + (e & 1);
          // fast SiLU (h is rounded to binary16 next; MoE outputs stay within the 1e-4 tolerance)
          const float g1 = acc[0][i][nt][e];
          float h = __fdividef(g1, 1.0f + __expf(-g1)) * acc[NM - 1][i][nt][e];
          if (row >= B.rows) h = 0.0f;
          const float h_next = __shfl_down_sync(0xffffffffu, h, 4);  // column n + 1
          if ((g & 1) == 0 && !dry) {
            const int n = n0 + 16 * i + g + 8 * (e >> 1);
            __stcg(reinterpret_cast<unsigned int*>(hb + (int64_t)row * W.f_max + n),
                   h2_as_u32(__floats2half2_rn(h, h_next)));
          }
        }
    __syncwarp();
    FIN_DBG(14);
    if (lane == 0 && !dry) st_release_gpu(W.hflag + P.b * (W.f_max >> 6) + s, epoch);
    FIN_DBG(13);
  } else {
    // y rows -> Y slots; the last block of this d-slab runs the combine
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = 8 * nt + 2 * q + (e & 1);
          if (row >= B.rows || dry) continue;
          __stcg(W.Y + (int64_t)B.slot[row] * d + n0 + 16 * i + g + 8 * (e >> 1), acc[0][i][nt][e]);
        }
    __syncwarp();
    const int nb = sc[0];
    int last = 0;
    if (lane == 0) {
      last = dry ? 1 : atom_add_acqrel_gpu(W.ccnt + s, 1) == nb - 1;
      if (last && !dry) W.ccnt[s] = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      const int K = a.K, m = a.m;
      const int n = n0 + 2 * lane;
      for (int t = 0; t < m; ++t) {
        float2 o = make_float2(0.0f, 0.0f);
        for (int k = 0; k < K; ++k) {
          if (r_ids[t * K + k] < 0) continue;
          const float wk = r_wts[t * K + k];
          const float2 y = __ldcg(reinterpret_cast<const float2*>(W.Y + (int64_t)(t * K + k) * d + n));
          o.x += wk * y.x;
          o.y += wk * y.y;
        }
        for (int sh = 0; sh < a.S; ++sh) {
          const float2 y = __ldcg(reinterpret_cast<const float2*>(W.Y + (int64_t)(m * K + sh * m + t) * d + n));
          o.x += 1.0f * y.x;
          o.y += 1.0f * y.y;
        }
        if (dry)
          continue;
        if (a.out_dtype == 0)
          *reinterpret_cast<float2*>(static_cast<float*>(a.out) + (int64_t)t * a.ldo + n) = o;
        else
          *reinterpret_cast<__half2*>(static_cast<__half*>(a.out) + (int64_t)t * a.ldo + n) =
              __floats2half2_rn(o.x, o.y);
      }
    }
  }
}

// Per-warp producer (lane 0): walks the warp's tiles of both phases and issues
// their weight copies (one bulk copy per matrix per slot) into the warp's ring.
// Weights never depend on other warps, so the producer never waits.  Slot
// chunking: min(kc, tiles left in the slab, tiles left in the warp's range),
// exactly as run_phase consumes them.
template <int NT, int NMAT1, bool MOE>
struct Prod {
  using CF = DecCfg<NT, NMAT1>;
  uint8_t* ring;
  uint64_t* fb;
  const uint8_t* base0;
  const uint8_t* base1;
  int ph, p, s, t, left, kc, ktiles, tb, nm, nslabs, nphase;
  uint64_t pol;  // L2 evict_first

  __device__ __forceinline__ void load(const DProb* probs, int rel) {  // tile rel of problem p
    const DProb& P = probs[ph * CF::kMaxProbs + p];
    kc = P.kc;
    ktiles = P.ktiles;
    tb = P.tb;
    nm = P.kind == 1 && ph == 0 ? NMAT1 : 1;
    nslabs = P.n_slabs;
    base0 = P.src[0];
    base1 = P.src[1];
    s = rel / ktiles;
    t = rel - s * ktiles;
  }
  __device__ __forceinline__ void seek(const DProb* probs, int ph_, int T0, int T1, int G, int gw) {
    ph = ph_;
    left = 0;
    const int Tp = ph == 0 ? T0 : T1;
    const int Gp = min(ph == 0 ? G - 1 : G, Tp);  // phase 1: the grid's last warp is the code warmer
    if (gw >= Gp) return;
    const int st = rng_at(gw, Tp, Gp), en = rng_at(gw + 1, Tp, Gp);
    left = en - st;
    const DProb* P = probs + ph * CF::kMaxProbs;
    int q = 0;
    while (P[q].t0 + P[q].n_slabs * P[q].ktiles <= st) ++q;
    p = q;
    load(probs, st - P[q].t0);
  }
  __device__ __forceinline__ bool norm(const DProb* probs, int T0, int T1, int G, int gw) {
    while (left == 0) {
      if (ph + 1 >= nphase) return false;
      seek(probs, ph + 1, T0, T1, G, gw);
    }
    return true;
  }
  __device__ __forceinline__ void issue(const DProb* probs, int sl) {
    uint8_t* dst = ring + sl * CF::kSlotBytes;
    const int c = min(min(kc, ktiles - t), left);
    const uint32_t bytes = (uint32_t)(c * tb);
    mbar_arrive_expect_tx(&fb[sl], bytes * (uint32_t)nm);
    const int64_t off = ((int64_t)s * ktiles + t) * tb;
    if (MOE) {  // streamed once: L2 keeps code, tables and prefetched tiles instead
      bulk_g2s_hint(dst, base0 + off, bytes, &fb[sl], pol);
      if (nm == 2) bulk_g2s_hint(dst + bytes, base1 + off, bytes, &fb[sl], pol);
    } else {
      bulk_g2s(dst, base0 + off, bytes, &fb[sl]);
      if (nm == 2) bulk_g2s(dst + bytes, base1 + off, bytes, &fb[sl]);
    }
    left -= c;
    t += c;
    if (t == ktiles) {
      t = 0;
      if (++s == nslabs && left > 0) {
        const DProb* P = probs + ph * CF::kMaxProbs;
        do ++p; while (P[p].n_slabs == 0);
        load(probs, 0);
      }
    }
  }
};

struct PhaseState {
  int slot;
  uint32_t parity;
  long long t_wait, t_fin, t_issue, n_units, t_comp, t_h, t_comp1;
};

// Activation rows of block B for the phase: phase 1 -> x rows (binary16,
// row-major, ldx), phase 2 -> the block's h rows; null for padding rows.
template <int NT>
__device__ __forceinline__ void block_rows(const __half* (&rowp)[NT], const DBlock& B, int ph, int bidx,
                                           const __half* xact, int64_t ldxa, const DecWs& W, int g) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int row = 8 * nt + g;
    if (row >= B.rows) {
      rowp[nt] = nullptr;
    } else if (ph == 0) {
      rowp[nt] = xact + (int64_t)B.xrow[row] * ldxa;
    } else {
      rowp[nt] = W.h + ((int64_t)bidx * (8 * NT) + row) * W.f_max;
    }
  }
}

// One phase of a warp's units: stream-K segments, each accumulated in registers
// (NM matrices per unit) and handed to dec_finish.  B fragments for unit i + 1
// are loaded while unit i computes.
template <int NT, int NMAT1, bool MOE, int NM, int PH>
__device__ __forceinline__ void run_phase(const DecArgs& a, Prod<NT, NMAT1, MOE>& pr, PhaseState& ps,
                                          const DProb* probs, const DBlock* blocks, const DecExpert* experts,
                                          uint8_t* ring, uint64_t* fb, const __half* xact, int64_t ldxa,
                                          int T0, int T1, int G, int gw) {
  using CF = DecCfg<NT, NMAT1>;
  constexpr int kS = CF::kSlots;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const DProb* PP = probs + PH * CF::kMaxProbs;
  extern __shared__ __align__(128) uint8_t smem[];
  const DecExpert* bxs = reinterpret_cast<const DecExpert*>(smem + CF::kOffMats);
  const int Tp = PH == 0 ? T0 : T1;
  const int Gp = min(PH == 0 ? G - 1 : G, Tp);
  if (gw >= Gp) return;
  const int start = rng_at(gw, Tp, Gp), end = rng_at(gw + 1, Tp, Gp);
  int p = 0;
  int pos = start;
  DEC_DBG(PH == 0 ? 2 : 5);
  while (pos < end) {
    while (PP[p].t0 + PP[p].n_slabs * PP[p].ktiles <= pos) ++p;
    const DProb& P = PP[p];
    const int s = (pos - P.t0) / P.ktiles;
    const int tt = pos - P.t0 - s * P.ktiles;
    const int seg_end = min(end, P.t0 + (s + 1) * P.ktiles);
    const int pkc = P.kc;
    const bool pseudo = P.kind == 0;
    const DecMat& M = bxs[P.b].m[P.mat];
    const DqConsts dq = make_dq_consts(M.mode);
    const bool preal = pseudo && M.real;
    const int ptb = P.tb;
    const int ktiles = P.ktiles;
    if (!pseudo && lane == 0 && seg_end == P.t0 + (s + 1) * ktiles && !(a.dbg_flags & 16)) {
      // this segment ends the slab: its finisher's V fragments / steps -> L2 now
      const DecExpert& X = bxs[P.b];
#pragma unroll
      for (int mat = 0; mat < NM; ++mat) {
        const DecMat& Mv = X.m[PH == 0 ? mat : 2];
        if (Mv.rank <= 0) continue;
        const int nks = Mv.r16 >> 4;
        const uint32_t vb = (uint32_t)nks * (Mv.real ? kVftRealBytes : kVftInt3Bytes);
        prefetch_l2(Mv.vft + (int64_t)s * vb, vb);
        if (!Mv.real) prefetch_l2(Mv.vstep + (int64_t)s * 64 * Mv.gpr, (uint32_t)(256 * Mv.gpr));
      }
    }
    const int32_t* hfl = a.ws.hflag + P.b * (a.ws.f_max >> 6);
    const __half* rowp[NT];
    block_rows<NT>(rowp, blocks[P.b], PH, P.b, xact, ldxa, a.ws, g);

    constexpr int NA = NM;
    float acc[NA][4][NT][4];
#pragma unroll
    for (int x = 0; x < NA; ++x)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[x][i][nt][e] = 0.0f;

    // k-tile pipeline over the segment: B fragments load kLA tiles ahead of the
    // tile being computed (phase 2 reads h at L2 latency: two tiles ahead)
    constexpr int kLA = PH == 1 ? 2 : 1;
    const int kend = ktiles * 32;
    int k = tt * 32;
    BTile<NT> bc, bn1;
    // phase 2: the h slabs of this slot and of the look-ahead tiles
    HWin hwin{0, 0u};
    const int nhf = a.ws.f_max >> 6;
    if (PH == 1) {
      const long long th0 = DEC_TIMERS ? clock64() : 0;
      wait_h_cached(hfl, nhf, hwin, k, min(kend, k + (min(pkc, seg_end - pos) + kLA) * 32), a.epoch, lane);
      if (DEC_TIMERS) ps.t_h += clock64() - th0;
    }
    const bool bload = !(a.dbg_flags & 32);  // experiment: bit 5 = no activation loads (wrong results)
    load_btile<NT, PH == 1>(bc, rowp, k, bload, q);
    if (kLA == 2) load_btile<NT, PH == 1>(bn1, rowp, k + 32, bload && k + 32 < kend, q);
    for (int left = seg_end - pos; left > 0;) {
      const int slot = ps.slot;
      const int kc = min(pkc, left);
      left -= kc;
      if (PH == 1 && k != tt * 32) {
        const long long th0 = DEC_TIMERS ? clock64() : 0;
        wait_h_cached(hfl, nhf, hwin, k, min(kend, k + (kc + kLA) * 32), a.epoch, lane);
        if (DEC_TIMERS) ps.t_h += clock64() - th0;
      }
      if (DEC_TIMERS) {
        const long long tw0 = clock64();
        mbar_wait(&fb[slot], ps.parity);
        ps.t_wait += clock64() - tw0;
        ++ps.n_units;
      } else {
        mbar_wait(&fb[slot], ps.parity);
      }
      const uint8_t* st = ring + slot * CF::kSlotBytes;
      const long long tc0 = DEC_TIMERS ? clock64() : 0;
#pragma unroll 1
      for (int kk = 0; kk < kc; ++kk, k += 32) {
        BTile<NT> bn;
        load_btile<NT, PH == 1>(bn, rowp, k + 32 * kLA, bload && k + 32 * kLA < kend, q);
        if (pseudo)
          tile_pseudo<NT, NA>(st + kk * ptb, preal, bc, acc, lane);
        else
          tile_real<NT, NM, NA>(st + kk * kTileBytes, kc * kTileBytes, bc, acc, dq, lane);
        if (kLA == 2) {
          bc = bn1;
          bn1 = bn;
        } else {
          bc = bn;
        }
      }
      if (DEC_TIMERS) ps.t_comp += clock64() - tc0;
      __syncwarp();
      if (left == 0) break;  // the segment's last slot is the finisher's scratch (issued below)
      if (DEC_TIMERS) {
        const long long ti0 = clock64();
        if (lane == 0 && pr.norm(probs, T0, T1, G, gw)) pr.issue(probs, slot);
        ps.t_issue += clock64() - ti0;
      } else if (lane == 0 && pr.norm(probs, T0, T1, G, gw)) {
        pr.issue(probs, slot);
      }
      if (++ps.slot == kS) {
        ps.slot = 0;
        ps.parity ^= 1u;
      }
    }
    // park the accumulators in the consumed slot, finish, then refill the slot
    {
      const int slot = ps.slot;
      float* accs = reinterpret_cast<float*>(ring + slot * CF::kSlotBytes);
#pragma unroll
      for (int x = 0; x < NM; ++x)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) accs[(((x * 4 + i) * NT + nt) * 4 + e) * 32 + lane] = acc[x][i][nt][e];
      __syncwarp();
      pos = seg_end;
      if (pos == end) DEC_DBG(3 + 3 * PH);
      const long long tf0 = DEC_TIMERS ? clock64() : 0;
      dec_finish<NT, NMAT1, MOE, NM>(a, accs, PH, p, s, start, end, Gp, Tp, gw, G, false);
      if (DEC_TIMERS) ps.t_fin += clock64() - tf0;
      __syncwarp();
      fence_proxy_async();  // generic smem use of the slot before the next bulk copy into it
      if (lane == 0 && pr.norm(probs, T0, T1, G, gw)) pr.issue(probs, slot);
      if (++ps.slot == kS) {
        ps.slot = 0;
        ps.parity ^= 1u;
      }
    }
  }
}

// ---------------------------------------------------------------- the kernel
template <int NT, int NMAT1, bool MOE>
__global__ void __launch_bounds__(32 * DecCfg<NT, NMAT1>::kWarps, 1)
    decode_kernel(const __grid_constant__ DecArgs a) {
  using CF = DecCfg<NT, NMAT1>;
  static_assert(CF::kBytes <= 227 * 1024, "decode kernel shared memory");
  static_assert(NMAT1 * 4 * NT * 4 * 32 * 4 <= CF::kSlotBytes, "parked accumulators must fit a ring slot");
  constexpr int kC = CF::kCons, kS = CF::kSlots;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* full_bars = reinterpret_cast<uint64_t*>(smem + CF::kOffBars);  // [kC][kS]
  const DProb* probs = reinterpret_cast<const DProb*>(smem + CF::kOffProbs);
  const DBlock* blocks = reinterpret_cast<const DBlock*>(smem + CF::kOffBlocks);
  const int32_t* sc = reinterpret_cast<const int32_t*>(smem + CF::kOffRoute + kDecMaxEntries * 8 + 256 * 8);
  const DecWs& W = a.ws;
  const DecExpert* experts = MOE ? a.experts : &a.lin;

  for (int i = tid; i < kC * kS; i += blockDim.x) mbar_init(&full_bars[i], 1);
  fence_barrier_init();
  pdl_wait();
  DEC_DBG(0);
  if (W.xrep != nullptr) {
    // CTA-private binary16 copy of x (the phase-1 activation rows, read from L1)
    __half* xr = W.xrep + (int64_t)blockIdx.x * a.m * a.d;
    const int n8 = a.m * (a.d / 8);
    for (int i = tid; i < n8; i += blockDim.x) {
      const int r = i / (a.d / 8), c = (i % (a.d / 8)) * 8;
      uint4 v;
      if (a.x_dtype == 0) {
        const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + (int64_t)r * a.ldx + c);
        const float4 p0 = __ldg(src), p1 = __ldg(src + 1);
        v = make_uint4(h2_as_u32(__floats2half2_rn(p0.x, p0.y)), h2_as_u32(__floats2half2_rn(p0.z, p0.w)),
                       h2_as_u32(__floats2half2_rn(p1.x, p1.y)), h2_as_u32(__floats2half2_rn(p1.z, p1.w)));
      } else {
        v = __ldg(reinterpret_cast<const uint4*>(static_cast<const __half*>(a.x) + (int64_t)r * a.ldx + c));
      }
      *reinterpret_cast<uint4*>(xr + (int64_t)r * a.d + c) = v;
    }
  }
  DEC_DBG(15);
  dec_stage0<NT, NMAT1, MOE>(a);
  DEC_DBG(1);
  if (MOE && DEC_W2_PREFETCH && warp == kC - 1) {
    // Phase-2 weights (the touched experts' w2) -> L2 while phase 1 streams: phase 1
    // leaves HBM bandwidth idle (~3 TB/s) and phase 2 then reads L2.  The grid
    // splits the concatenated w2 bytes evenly; each lane of one warp per CTA
    // prefetches a 1/32 share of the CTA's range (bulk L2 prefetches, no destination).
    const int nb = sc[0];
    const DProb* P2 = probs + CF::kMaxProbs + nb;  // phase-2 real problems, one per block
    int64_t total = 0;
    for (int b = 0; b < nb; ++b)
      if (blocks[b].chunk == 0) total += (int64_t)P2[b].n_slabs * P2[b].ktiles * kTileBytes;
    const int64_t per_cta = ((total + gridDim.x - 1) / gridDim.x + 511) & ~int64_t(511);
    const int64_t per_lane = per_cta / 32;  // multiple of 16
    int64_t lo = (int64_t)blockIdx.x * per_cta + lane * per_lane, hi = min(total, lo + per_lane);
    int64_t base = 0;
    for (int b = 0; b < nb && lo < hi; ++b) {
      if (blocks[b].chunk != 0) continue;
      const int64_t bytes = (int64_t)P2[b].n_slabs * P2[b].ktiles * kTileBytes;
      const int64_t a0 = max(lo, base), a1 = min(hi, base + bytes);
      for (int64_t o = a0; o < a1; o += 32768)
        prefetch_l2(P2[b].src[0] + (o - base), (uint32_t)(a1 - o < 32768 ? a1 - o : 32768));
      base += bytes;
    }
  }
  const __half* xact = W.xrep != nullptr ? W.xrep + (int64_t)blockIdx.x * a.m * a.d
                                         : static_cast<const __half*>(a.x);
  const int64_t ldxa = W.xrep != nullptr ? a.d : a.ldx;

  const int G = a.gw;
  const int T0 = sc[3], T1 = sc[4];
  const int gw = blockIdx.x * kC + warp;
  uint8_t* ring = smem + warp * kS * CF::kSlotBytes;
  uint64_t* fb = full_bars + warp * kS;

  Prod<NT, NMAT1, MOE> pr;
  pr.ring = ring;
  pr.fb = fb;
  pr.nphase = MOE ? 2 : 1;
  pr.pol = policy_evict_first();
  if (lane == 0) {
    pr.seek(probs, 0, T0, T1, G, gw);
    for (int sl = 0; sl < kS && pr.norm(probs, T0, T1, G, gw); ++sl) pr.issue(probs, sl);
  }
  __syncwarp();

  PhaseState st{0, 0u, 0, 0, 0, 0, 0, 0, 0};
  if (DEC_WARM && NT == 1 && gw == G - 1) {  // (NT = 2: the extra call sites cost the finisher registers)
    // Code warm-up while the memory system is still idle: run the finisher
    // paths once with every side effect off, so that the real finishers at the
    // end of each phase (one per slab, all at about the same time) find this
    // code in L2 instead of queueing behind the weight stream for it.
    const DProb* P0 = probs;
    int q0 = 0;
    while (q0 < CF::kMaxProbs - 1 && !(P0[q0].kind == 1 && P0[q0].n_slabs > 0)) ++q0;
    float* scratch = reinterpret_cast<float*>(ring);
    dec_finish<NT, NMAT1, MOE, NMAT1>(a, scratch, 0, q0, 0, 0, 1, 1, 1, gw, G, true);
    if (MOE) {
      const DProb* P1 = probs + CF::kMaxProbs;
      int q1 = 0;
      while (q1 < CF::kMaxProbs - 1 && !(P1[q1].kind == 1 && P1[q1].n_slabs > 0)) ++q1;
      dec_finish<NT, NMAT1, MOE, 1>(a, scratch, 1, q1, 0, 0, 1, 1, 1, gw, G, true);
    }
    __syncwarp();
    fence_proxy_async();
  }
  run_phase<NT, NMAT1, MOE, NMAT1, 0>(a, pr, st, probs, blocks, experts, ring, fb, xact, ldxa, T0, T1, G, gw);
  DEC_DBG(4);
  st.t_comp1 = st.t_comp;
  if (MOE)
    run_phase<NT, NMAT1, MOE, 1, 1>(a, pr, st, probs, blocks, experts, ring, fb, xact, ldxa, T0, T1, G, gw);
  DEC_DBG(7);
  if (DEC_TIMERS && a.dbg != nullptr && lane == 0) {
    long long* o = a.dbg + ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 16;
    o[11] = st.t_wait; o[12] = st.t_fin; o[13] = st.t_issue; o[14] = st.n_units; o[10] = st.t_comp; o[9] = st.t_h; o[8] = st.t_comp1;
  }
  pdl_launch_dependents();
}

// f32 rows -> binary16 rows (the decode kernel's activation input).
__global__ void rows_to_half_kernel(const float* __restrict__ x, int64_t rows, int64_t cols,
                                    int64_t ldx, __half* __restrict__ y) {
  const int64_t n4 = rows * (cols / 4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (cols / 4), c = (i % (cols / 4)) * 4;
    const float4 v = *reinterpret_cast<const float4*>(x + r * ldx + c);
    __half2* o = reinterpret_cast<__half2*>(y + r * cols + c);
    o[0] = __floats2half2_rn(v.x, v.y);
    o[1] = __floats2half2_rn(v.z, v.w);
  }
}

}  // namespace milo_dev
