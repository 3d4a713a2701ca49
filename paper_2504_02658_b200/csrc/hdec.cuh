// K4: the decode-regime MoE layer as an "h-local" persistent kernel.
//
// Reference semantics per matrix: milo::gemm_w3a16 (proj/src/gemm.cpp:117-199),
//   C = half(A) * dequant(W) + (half(A) U) V   (fp32 accumulation),
// composed into the routed expert layer of SURVEY.md section 8b (the reference
// has no MoE layer; oracle/milo_oracle.c defines the composition):
//   h_e = half(silu(x W1_e + t1 V1_e) * (x W3_e + t3 V3_e)),  y_e = h_e W2_e + t2 V2_e,
//   out[t] = sum_k w[t,k] y_{e(t,k)}[t] + sum_shared y_s[t].
//
// Why "h-local": w2 reduces over f, so the 64 h values of one f-slab c of an
// expert are all that slab c's rows of W2 need.  A UNIT = (expert, f-slab c) =
//   P1: the W1 and W3 columns of slab c over all d (-> its 64 h values), then
//   P2: the W2 rows of slab c over all d (-> their share of every output).
// Units never wait for each other: no phase barrier, no h round trip through
// HBM.  The grid's CTAs split the concatenated units' work ("pairs": one P1
// k-step = a W1 and a W3 macro tile, one P2 d-slab = 2 W2 tiles, 1792 B each)
// into equal ranges (stream-K).  A unit cut by a range boundary is finished by
// the CTA holding the END of its P1 (the "tail holder"): lower CTAs publish P1
// partials, a CTA holding only a P2 tail reads the published h.  Each CTA does
// the piece straddling its range END first and the one straddling its START
// last, so every cross-CTA value is produced at the start of one CTA's run and
// consumed at the end of another's.
//
// P2 contributions go straight into the output with fp32 vector reductions
// (red.global.add.v4.f32) scaled by the routing weight; the grid zeroes the
// output first.  LoRC: t = x U per (expert, w1|w3) comes from small "T items"
// at the start (tagged partials, summed in a fixed order); t V of slab c is
// added by the tail holder before SwiGLU; t2 = h U2 is accumulated per unit
// (fp32 reductions, a counter per expert); t2 V2 is done by "V2 items" at the
// end, once the expert's counter is complete.
//
// CTA = 8 consumer warps + 1 producer warp.  The producer alone walks the
// event sequence: it streams each event's bytes (weights, compensator tiles and
// the x rows the event multiplies) with 1D bulk copies into a ring of 37 KB
// stages (copies issued by up to 32 lanes in parallel: one thread serialises
// its bulk copies at ~300 cycles each, tools/micro/bulk_issue.cu) and publishes
// a 16-byte descriptor per stage, with the consumer-only steps (reductions,
// SwiGLU, publications, waits) folded in as flags.  Consumers split each
// stage's tiles over the warps, de-quantize in registers bit-exactly
// (layout.cuh) and run mma.m16n8k16 with W^T as the A operand; every operand
// they touch is in shared memory.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "decode.cuh"

namespace milo_dev {

constexpr int kHdProd = 2;                      // producer warps (alternate stages)
constexpr int kHdMaxParts = 72;                 // participating experts per launch
constexpr int kHdMaxTok = 16;                   // tokens per expert (NT <= 2)
constexpr int kHdCtrl = 4 + kHdMaxParts;        // per-parity control ints
constexpr int kHdTK = 16;                       // U pseudo tiles per T item
constexpr int kHdV2K = 8;                       // V2 rank steps per V2 item
constexpr int kHdScr = 68;                      // epilogue scratch row stride (floats)
constexpr int kHdDbgG = 1024;                   // timeline layout: regions sized for this many CTAs

// Per-expert static view (host-built, 16 B).
struct HdExp {
  int32_t nu, kt2;     // f / 64, f / 32
  int8_t nks[3];       // compensator rank steps (16 ranks) of w1, w3, w2 (0: none)
  int8_t gpr[3];       // 64-rank step groups of w1, w3, w2
  int8_t mode, pad;
};

struct HdArgs {
  int32_t m, E, K, S, score_mode, d;
  const float* logits;   // m x E, or null: routing given
  const int32_t* ids_in;
  const float* wts_in;
  int32_t* ids_out;      // optional routing outputs (logits given)
  float* wts_out;
  const DecExpert* experts;  // E routed then S shared
  const HdExp* hexp;
  const uint8_t* w2maps;  // per expert: a 128-byte TMA map of W2's slab-major tiles (boxes of 8 slabs x 2 k-tiles)
  const __half* x;       // binary16 rows, ld = ldx
  int64_t ldx;
  void* out;
  int32_t out_dtype;     // 0 f32 (accumulated in place), 1 f16 (via acc)
  int64_t ldo;
  int32_t epoch;
  int32_t* ctrl;         // this call's control block [kHdCtrl] (zero at entry)
  int32_t* ctrl_next;    // the other parity's block: zeroed by this call for the next
  uint64_t* tpart;       // [T items][16 tok][16 ranks] tagged
  uint64_t* part;        // [grid][1024 NT] tagged P1 partials
  uint64_t* hpub;        // [grid][16 tok][32] tagged h pairs
  float* t2acc;          // fp32, zeroed by the kernel
  float* acc;            // f16 output: fp32 accumulator m x d (zeroed by the kernel)
  long long* dbg;       // optional timeline: [grid][128] consumer warp 0, then [grid][64] producer stamps
  int32_t dbg_flags;    // experiments: bit 0 no output reductions, bit 1 no P2 epilogue, bit 2 no copies, bit 4 producers alone (no copies, no waits), bit 5 no P1 compute, bit 6 no L2 prefetch, bit 7 no P2 compute
};

struct HPart {
  int32_t e, rows, nu, u0;     // expert, tokens, units (f / 64), first unit
  int32_t t2off, tb, vb, kt2;  // t2 accumulator offset (floats), first T item, first V2 item, f / 32
  int8_t nks[3];               // rank steps of w1, w3, w2
  int8_t gpr[3];
  int8_t mode, ksp;            // de-quant mode; P1 k-steps per stage
  int8_t xrow[kHdMaxTok];
  float wt[kHdMaxTok];
};
static_assert(sizeof(HPart) <= 128, "HPart");

// Ring descriptor (one per stage).
struct HDesc {
  uint8_t type, flags, j, n;
  uint16_t c, a;
  uint8_t mat, pad;
  uint16_t aux, head, tail;
};
static_assert(sizeof(HDesc) == 16, "HDesc");
enum : uint8_t {
  F_FIRST = 1,      // P1: first stage of the piece (zero the accumulators)
  F_HEADPUB = 2,    // after: reduce + publish the piece's P1 partial
  F_FINBEGIN = 4,   // after: reduce + add the lower CTAs' partials -> ybuf
  F_FINH = 8,       // after: SwiGLU -> h
  F_PUBH = 16,      //        ... and publish h
  F_T2DONE = 32,    // after: count the unit's t2 contribution
  F_HWAIT = 64,     // before: read h published by CTA `tail`
  F_END = 128,
};

// Ring geometry per token-tile count (12 consumer warps at 128 registers measured
// slower than 8 at 168: 1.31 us per 24-tile stage vs 1.47 us per 32).
template <int NT>
struct HdCfg {
  // NT = 1: 12 consumer warps (3 per SM sub-partition: at 2 the de-quantization stalls on
  // its own latencies) in 152 registers after setmaxnreg (the producer warpgroup drops to
  // 40), three 48.5 KB stages; NT = 2: 8 consumer warps, four 37 KB stages.
  static constexpr int kCtasPerSm = 1;
  static constexpr int kCons = NT == 1 ? 12 : 8;       // consumer warps
  static constexpr bool kSetMaxNreg = NT == 1;         // producer warpgroup (4 warps: 2 producers, 2 idle)
  static constexpr int kConsRegs = 152, kProdRegs = 40;
  static constexpr int kThreads = 32 * (kCons + (kSetMaxNreg ? 4 : kHdProd));
  static constexpr int kStage = NT == 1 ? 49664 : 37888;  // ring stage bytes
  static constexpr int kNS = NT == 1 ? 3 : 4;          // ring stages
  static constexpr int kP2 = NT == 1 ? 24 : 16;        // P2 d-slabs per stage
  // P1 k-steps per stage for `rows` tokens (multiples of the consumer warps)
  static __device__ __forceinline__ int ksp(int rows) {
    return NT == 1 ? (rows <= 4 ? 24 : 12) : (rows <= 8 ? 16 : 8);
  }
  static constexpr int kFV = (kStage - 2048) / 1024 < 32 ? (kStage - 2048) / 1024 : 32;  // V rank steps per FIN-V stage
  static constexpr int kFU = kStage / 1280;            // U2 rank groups per FIN-U stage
  static constexpr int kOffRing = 0;
  static constexpr int kOffRed = kNS * kStage;
  static constexpr int kScrBytes = 0;                                          // (epilogues shuffle in registers)
  static constexpr int kTreeBytes = 4 * 32 * NT * 32 * 4;                      // P1 reduction: 4 slots
  static constexpr int kFvBytes = 8 * NT * (16 * kFV + 8) * 4;                // FIN-V t image
  static constexpr int kRed0 = kScrBytes + 8 * NT * (16 * kHdV2K + 8) * 4;    // + V2's t2 image
  static constexpr int kRedBytes = kRed0 > kTreeBytes ? (kRed0 > kFvBytes ? kRed0 : kFvBytes)
                                                      : (kTreeBytes > kFvBytes ? kTreeBytes : kFvBytes);
  static constexpr int kOffY = kOffRed + kRedBytes;             // [2][4][NT][4][32] f32
  static constexpr int kOffH = kOffY + 2 * 4 * NT * 4 * 32 * 4;  // [16][72] f16
  static constexpr int kOffParts = kOffH + kHdMaxTok * 72 * 2;
  static constexpr int kOffTc = kOffParts + kHdMaxParts * 128;    // t cache [2][8 NT][72] f32 (ranks <= 64)
  static constexpr int kOffPend = kOffTc + 2 * 8 * NT * 72 * 4;      // deferred t2 counts [kHdMaxParts] i16
  static constexpr int kOffDesc = kOffPend + kHdMaxParts * 2;
  static constexpr int kOffBars = kOffDesc + kNS * 16;           // full[NS], empty[NS]
  static constexpr int kOffMisc = kOffBars + 2 * kNS * 8;
  static constexpr int kOffDq = kOffMisc + 64;   // DqConsts for modes 0, 1
  static constexpr int kBytes = kOffDq + 64;
};

enum : int {
  EV_T = 1, EV_P1, EV_HEADPUB, EV_FINBEGIN, EV_FV, EV_FINH, EV_FU, EV_T2DONE, EV_HWAIT, EV_P2, EV_V2
};

struct HEv {
  int type, j, c, a, n, mat, aux;  // aux: P1 first flag / FINBEGIN first head CTA / HWAIT tail CTA /
                                   // FINH publish flag / V2 rank-step start; V2: c = first d-slab, n = slabs, mat = steps
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_b64(const uint64_t* p) {
  uint64_t a;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
  return a;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
template <int NT>
__device__ __forceinline__ void cons_bar() { named_bar_sync(1, 32 * HdCfg<NT>::kCons); }

// The grid's split of the unit pairs: CTA i holds [lo(i), lo(i + 1)).  CTAs that also
// run a T item (round-robin from CTA 0) or a V2 item (round-robin from CTA G - 1) get
// kHdTCost / kHdVCost fewer pairs, so the grid still finishes together:
//   lo(i) = floor(i (Tot + X nT + Y nV) / G) - X T(i) - Y V(i),
// T(i), V(i) = the T / V2 items owned by CTAs below i.
constexpr int kHdTCost = 0, kHdVCost = 0;  // pairs (one pair ~ 1792 B of weights); 40 / 30 measured no better (noise-level)
struct HRange {
  long long Tot, Sum;
  int G, nT, nV, X, Y;
  __device__ __forceinline__ void init(long long tot, int g, int nt, int nv) {
    Tot = tot;
    G = g;
    nT = nt;
    nV = nv;
    const long long R = (tot + g - 1) / g;
    X = (int)(R / 4 < kHdTCost ? R / 4 : kHdTCost);
    Y = (int)(R / 4 < kHdVCost ? R / 4 : kHdVCost);
    Sum = tot + (long long)X * nt + (long long)Y * nv;
  }
  __device__ __forceinline__ long long lo(int i) const {
    if (i >= G) return Tot;
    const long long t = (long long)(nT / G) * i + min(i, nT % G);
    const long long v = (long long)(nV / G) * i + max(0, nV % G - G + i);
    const long long r = (long long)i * Sum / G - (long long)X * t - (long long)Y * v;
    return r < 0 ? 0 : (r > Tot ? Tot : r);
  }
  __device__ __forceinline__ int owner(long long x) const {  // the CTA whose range holds pair x
    int a = 0, b = G - 1;
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (lo(mid) <= x) a = mid; else b = mid - 1;
    }
    return a;
  }
};

// B fragments of 32 k from a binary16 [row][.] image in shared memory (row
// stride rs halves, rows >= nrows read as zero) at column kb.
template <int NT>
__device__ __forceinline__ void load_bs(BTile<NT>& b, const __half* base, int rs, int nrows, int kb, int g, int q) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int r = 8 * nt + g;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint32_t b0 = 0u, b1 = 0u;
      if (r < nrows) {
        const __half* p = base + r * rs + kb + 16 * j + 2 * q;
        b0 = *reinterpret_cast<const uint32_t*>(p);
        b1 = *reinterpret_cast<const uint32_t*>(p + 8);
      }
      b.v[j][nt][0] = b0;
      b.v[j][nt][1] = b1;
    }
  }
}

// The producer's register copy of one expert's device pointers (reloaded when
// the participant changes: a dependent global load per stage would cost an L2
// round trip, ~1 us under the weight stream).
struct HMats {
  const uint8_t* w2map;
  const uint8_t* w[3];
  const uint8_t* upt[3];
  const uint8_t* vft[3];
  const float* vstep[3];
  int gpr[3];
  __device__ __forceinline__ void load(const DecExpert& X, const uint8_t* map) {
    w2map = map;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      w[i] = X.m[i].w;
      upt[i] = X.m[i].upt;
      vft[i] = X.m[i].vft;
      vstep[i] = X.m[i].vstep;
      gpr[i] = X.m[i].gpr;
    }
  }
};

// Copies of a copy event: count, and copy i (src, bytes, destination offset).
struct HCopy {
  const uint8_t* src;  // 1D: bytes; TMA (tma != 0): the tensor map, box at (x, y)
  uint32_t bytes, dst;
  int tma, x, y;
};
constexpr int kW2Box = 8;  // slabs per W2 TMA box (box = 8 slabs x 1792 B = 14336 B)
__device__ __forceinline__ int ev_ncopies(const HEv& ev, const HPart& P) {
  switch (ev.type) {
    case EV_T: return 1 + P.rows;
    case EV_P1: return 2 + P.rows;
    case EV_FV: return 2;
    case EV_FU: return ev.n;
    case EV_P2: return (ev.n + kW2Box - 1) / kW2Box;
    case EV_V2: return ev.n + 1;
    default: return 0;
  }
}
__device__ __forceinline__ uint32_t ev_bytes(const HEv& ev, const HPart& P) {
  switch (ev.type) {
    case EV_T: return ev.n * (kPseudoInt3Bytes + 64 * P.rows);
    case EV_P1: return ev.n * (2 * kTileBytes + 64 * P.rows);
    case EV_FV: return ev.n * kVftInt3Bytes + 256 * P.gpr[ev.mat];
    case EV_FU: return ev.n * 2 * kPseudoInt3Bytes;
    case EV_P2: return (ev.n + kW2Box - 1) / kW2Box * kW2Box * 2 * kTileBytes;
    case EV_V2: return ev.n * (ev.mat * kVftInt3Bytes + 256 * P.gpr[2]);
    default: return 0;
  }
}
// x rows (binary16) of k-tiles [k0, k0 + n) at offset xo of the stage, row stride n * 64 + 16 B.
__device__ __forceinline__ HCopy x_copy(const HdArgs& a, const HPart& P, int r, int k0, int n, uint32_t xo) {
  HCopy c{};
  c.src = reinterpret_cast<const uint8_t*>(a.x + (int64_t)P.xrow[r] * a.ldx + (int64_t)k0 * 32);
  c.bytes = n * 64;
  c.dst = xo + r * (n * 64 + 16);
  return c;
}
__device__ __forceinline__ HCopy ev_copy(const HdArgs& a, const HMats& X, const HEv& ev, const HPart& P, int KT,
                                         int i) {
  HCopy c{nullptr, 0u, 0u, 0, 0, 0};
  switch (ev.type) {
    case EV_T: {
      if (i > 0) return x_copy(a, P, i - 1, ev.a, ev.n, ev.n * kPseudoInt3Bytes);
      c.src = X.upt[ev.mat] + ((int64_t)ev.c * KT + ev.a) * kPseudoInt3Bytes;
      c.bytes = ev.n * kPseudoInt3Bytes;
      break;
    }
    case EV_P1: {
      if (i > 1) return x_copy(a, P, i - 2, ev.a, ev.n, 2 * ev.n * kTileBytes);
      c.src = X.w[i] + ((int64_t)ev.c * KT + ev.a) * kTileBytes;
      c.bytes = ev.n * kTileBytes;
      c.dst = i * ev.n * kTileBytes;
      break;
    }
    case EV_FV: {
      const int nks = P.nks[ev.mat];
      if (i == 0) {
        c.src = X.vft[ev.mat] + ((int64_t)ev.c * nks + ev.a) * kVftInt3Bytes;
        c.bytes = ev.n * kVftInt3Bytes;
      } else {
        c.src = reinterpret_cast<const uint8_t*>(X.vstep[ev.mat] + (int64_t)ev.c * 64 * X.gpr[ev.mat]);
        c.bytes = 256 * X.gpr[ev.mat];
        c.dst = ev.n * kVftInt3Bytes;
      }
      break;
    }
    case EV_FU: {
      c.src = X.upt[2] + ((int64_t)(ev.a + i) * P.kt2 + 2 * ev.c) * kPseudoInt3Bytes;
      c.bytes = 2 * kPseudoInt3Bytes;
      c.dst = i * 2 * kPseudoInt3Bytes;
      break;
    }
    case EV_P2: {  // box i: slabs [a + 8 i, a + 8 i + 8), k-tiles 2c, 2c + 1 (u64 column 224 c)
      c.src = X.w2map;
      c.tma = 1;
      c.x = 224 * ev.c;
      c.y = ev.a + kW2Box * i;
      c.bytes = kW2Box * 2 * kTileBytes;
      c.dst = i * kW2Box * 2 * kTileBytes;
      break;
    }
    case EV_V2: {
      const int nks = P.nks[2];
      if (i < ev.n) {
        c.src = X.vft[2] + ((int64_t)(ev.c + i) * nks + ev.aux) * kVftInt3Bytes;
        c.bytes = ev.mat * kVftInt3Bytes;
        c.dst = i * ev.mat * kVftInt3Bytes;
      } else {
        c.src = reinterpret_cast<const uint8_t*>(X.vstep[2] + (int64_t)ev.c * 64 * X.gpr[2]);
        c.bytes = ev.n * 256 * X.gpr[2];
        c.dst = ev.n * ev.mat * kVftInt3Bytes;
      }
      break;
    }
    default: break;
  }
  return c;
}

// ------------------------------------------------------------------ consumer pieces
// out (or the f16 path's accumulator) += wt[tok] * acc for up to two 64-column d-slabs
// (S0 from acc[0], S1 from acc[1] when `two`): scattered to the warp's scratch as
// [slab][tok][64], then 16-byte reductions.
template <int NT>
__device__ __forceinline__ void hd_epi_slab(const HdArgs& a, const HPart& P, const float (&acc)[4][NT][4], int S,
                                            int lane) {
  const int g = lane >> 2, q = lane & 3;
  float* dst = a.out_dtype == 0 ? static_cast<float*>(a.out) : a.acc;
  const int64_t ld = a.out_dtype == 0 ? a.ldo : a.d;
  if (P.rows <= 2) {  // decode: reductions straight from the fragments (lanes q == 0 hold tokens 0, 1)
    if (q == 0 && !(a.dbg_flags & 1)) {
#pragma unroll
      for (int tk = 0; tk < 2; ++tk) {
        if (tk >= P.rows) break;
        float* row = dst + (int64_t)P.xrow[tk] * ld + S * 64 + g;
        const float w = P.wt[tk];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          red_add_f32(row + 16 * i, w * acc[i][0][tk]);
          red_add_f32(row + 16 * i + 8, w * acc[i][0][2 + tk]);
        }
      }
    }
    return;
  }
  // 4 consecutive columns (lanes g .. g + 3 of one q) gathered into lanes g % 4 == 0,
  // then one 16-byte reduction per (column quad, token)
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float v = acc[i][nt][e];
        const float v1 = __shfl_down_sync(0xffffffffu, v, 4);
        const float v2 = __shfl_down_sync(0xffffffffu, v, 8);
        const float v3 = __shfl_down_sync(0xffffffffu, v, 12);
        const int tok = 8 * nt + 2 * q + (e & 1), n = 16 * i + g + 8 * (e >> 1);
        if ((g & 3) == 0 && tok < P.rows && !(a.dbg_flags & 1)) {
          const float w = P.wt[tok];
          red_add_v4(dst + (int64_t)P.xrow[tok] * ld + S * 64 + n, make_float4(w * v, w * v1, w * v2, w * v3));
        }
      }
}

__device__ __forceinline__ void wait_count(const int32_t* p, int v) {
  if (ld_acquire_gpu(p) >= v) return;
  const long long t0 = clock64();
  while (ld_acquire_gpu(p) < v) {
    __nanosleep(64);
    if (clock64() - t0 > 4000000000LL) __trap();
  }
}
// Waits for a tagged word of this call's epoch; returns its low 32 bits.
__device__ __forceinline__ uint32_t wait_tagged(const uint64_t* p, int epoch) {
  uint64_t w = ld_relaxed_b64(p);
  if ((uint32_t)(w >> 32) != (uint32_t)epoch) {
    const long long t0 = clock64();
    do {
      warp_backoff(t0);
      w = ld_relaxed_b64(p);
    } while ((uint32_t)(w >> 32) != (uint32_t)epoch);
  }
  return (uint32_t)w;
}

// acc[2][4][NT][4] as a flat array: element x -> ((mat * 4 + i) * NT + nt) * 4 + e
template <int NT>
__device__ __forceinline__ float& accel(float (&acc)[2][4][NT][4], int x) {
  return acc[x / (16 * NT)][(x / (4 * NT)) % 4][(x / 4) % NT][x % 4];
}

// ------------------------------------------------------------------ the kernel
template <int NT>
__global__ void __launch_bounds__(HdCfg<NT>::kThreads, HdCfg<NT>::kCtasPerSm) hdec_kernel(const __grid_constant__ HdArgs a) {
  using CF = HdCfg<NT>;
  constexpr int kHdCons = CF::kCons, kHdThreads = CF::kThreads, kHdStage = CF::kStage;
  constexpr int kCT = 32 * kHdCons;  // consumer threads
  constexpr int NS = CF::kNS;
  constexpr int kAcc = 32 * NT;  // accumulator values per lane of a P1 piece
  static_assert(CF::kBytes * CF::kCtasPerSm <= (CF::kCtasPerSm == 1 ? 227 * 1024 : 226 * 1024), "hdec shared memory");
  static_assert(NT != 1 || (24 * (2 * kTileBytes + 4 * 64) + 4 * 16 <= kHdStage && 12 * (2 * kTileBytes + 8 * 64) + 8 * 16 <= kHdStage), "P1 stage");
  static_assert(NT != 2 || (16 * (2 * kTileBytes + 8 * 64) + 8 * 16 <= kHdStage && 8 * (2 * kTileBytes + 16 * 64) + 16 * 16 <= kHdStage), "P1 stage");
  static_assert(CF::kP2 * 2 * kTileBytes <= kHdStage, "P2 stage");
  static_assert(kHdTK * kPseudoInt3Bytes + 8 * NT * (kHdTK * 64 + 16) <= kHdStage, "T stage");
  static_assert(CF::kFV * kVftInt3Bytes + 2048 <= kHdStage && CF::kFU * 2 * kPseudoInt3Bytes <= kHdStage, "FIN stages");
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int G = gridDim.x, cta = blockIdx.x;
  uint8_t* ring = smem + CF::kOffRing;
  float* red = reinterpret_cast<float*>(smem + CF::kOffRed);
  float* ybuf = reinterpret_cast<float*>(smem + CF::kOffY);
  __half* hbuf = reinterpret_cast<__half*>(smem + CF::kOffH);
  HPart* parts = reinterpret_cast<HPart*>(smem + CF::kOffParts);
  HDesc* desc = reinterpret_cast<HDesc*>(smem + CF::kOffDesc);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::kOffBars);
  uint64_t* empty = full + NS;
  int32_t* misc = reinterpret_cast<int32_t*>(smem + CF::kOffMisc);
  float* tcache = reinterpret_cast<float*>(smem + CF::kOffTc);
  int16_t* pend = reinterpret_cast<int16_t*>(smem + CF::kOffPend);
  const int m = a.m, E = a.E, K = a.K, d = a.d, KT = d / 32;
  long long* dbg = a.dbg != nullptr ? a.dbg + (int64_t)cta * 128 : nullptr;
  if (dbg != nullptr && tid == 0) dbg[0] = globaltimer();

  if (tid < NS) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], kHdCons);
  }
  fence_barrier_init();

  // ---------------- stage 0: routing and the participant table (every CTA)
  int32_t* r_ids = reinterpret_cast<int32_t*>(red);        // [16 * 16]
  float* r_wts = red + 256;                                  // [16 * 16]
  uint32_t* emask = reinterpret_cast<uint32_t*>(red + 512);  // [256] token bits per expert
  for (int e = tid; e < 256; e += kHdThreads) emask[e] = 0u;
  for (int j = tid; j < kHdMaxParts; j += kHdThreads) pend[j] = 0;
  if (K > 0) {
    if (a.logits != nullptr) {
      for (int t = warp; t < m; t += kHdThreads / 32)
        topk_regs(a.logits + (int64_t)t * E, E, K, a.score_mode, r_ids + t * K, r_wts + t * K, lane);
    } else {
      for (int i = tid; i < m * K; i += kHdThreads) {
        r_ids[i] = a.ids_in[i];
        r_wts[i] = a.wts_in[i];
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < m * K; i += kHdThreads) {
    const int e = r_ids[i];
    if (e >= 0 && e < E) atomicOr(&emask[e], 1u << (i / K));
    if (cta == 0 && a.logits != nullptr && a.ids_out != nullptr) {
      a.ids_out[i] = e;
      a.wts_out[i] = r_wts[i];
    }
  }
  __syncthreads();
  if (warp == 0) {  // participants: touched routed experts ascending, then the shared experts
    const int nse = E + a.S;
    const int nch = (KT + kHdTK - 1) / kHdTK;
    int np = 0, u = 0, t2 = 0, tb = 0, vb = 0;
    for (int e0 = 0; e0 < nse; e0 += 32) {
      const int e = e0 + lane;
      const int cnt = e < E ? __popc(emask[e]) : (e < nse ? m : 0);
      const bool on = cnt > 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, on);
      const int j = np + __popc(bal & ((1u << lane) - 1u));
      int nu = 0, nt2 = 0, ntb = 0, nvb = 0;
      if (on && j < kHdMaxParts) {
        const HdExp X = a.hexp[e];
        HPart& P = parts[j];
        P.e = e;
        P.rows = cnt;
        nu = X.nu;
        P.nu = nu;
        P.kt2 = X.kt2;
        P.mode = X.mode;
        P.ksp = (int8_t)CF::ksp(cnt);
        for (int mt = 0; mt < 3; ++mt) {
          P.nks[mt] = X.nks[mt];
          P.gpr[mt] = X.gpr[mt];
        }
        const int nks2 = X.nks[2];
        nt2 = cnt * 16 * nks2;
        ntb = (X.nks[0] + X.nks[1]) * nch;
        if (nks2 > 0) {
          if (nks2 <= kHdV2K) {
            const int ns = max(1, min(16, kHdStage / (nks2 * 1024 + 256 * X.gpr[2])));
            nvb = (d / 64 + ns - 1) / ns;
          } else {
            nvb = (d / 64) * ((nks2 + kHdV2K - 1) / kHdV2K);
          }
        }
        // token list (ascending) and combine weights
        int r = 0;
        for (int t = 0; t < m; ++t) {
          float w = 1.0f;
          if (e < E) {
            if (!(emask[e] >> t & 1u)) continue;
            for (int k = 0; k < K; ++k)
              if (r_ids[t * K + k] == e) w = r_wts[t * K + k];
          }
          P.xrow[r] = (int8_t)t;
          P.wt[r] = w;
          ++r;
        }
      }
      // exclusive prefix sums of units, t2 floats, T items, V2 items
      int iu = nu, i2 = nt2, it = ntb, iv = nvb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a0 = __shfl_up_sync(0xffffffffu, iu, o), a1 = __shfl_up_sync(0xffffffffu, i2, o);
        const int a2 = __shfl_up_sync(0xffffffffu, it, o), a3 = __shfl_up_sync(0xffffffffu, iv, o);
        if (lane >= o) {
          iu += a0;
          i2 += a1;
          it += a2;
          iv += a3;
        }
      }
      if (on && j < kHdMaxParts) {
        parts[j].u0 = u + iu - nu;
        parts[j].t2off = t2 + i2 - nt2;
        parts[j].tb = tb + it - ntb;
        parts[j].vb = vb + iv - nvb;
      }
      u += __shfl_sync(0xffffffffu, iu, 31);
      t2 += __shfl_sync(0xffffffffu, i2, 31);
      tb += __shfl_sync(0xffffffffu, it, 31);
      vb += __shfl_sync(0xffffffffu, iv, 31);
      np += __popc(bal);
    }
    if (lane == 0) {
      misc[0] = min(np, kHdMaxParts);
      misc[1] = u;
      misc[2] = t2;
      misc[3] = tb;
      misc[4] = vb;
    }
  }
  __syncthreads();
  const int np = misc[0], U = misc[1], t2tot = misc[2], nT = misc[3], nV = misc[4];
  // zero this call's accumulators (output / t2) and the next call's control block
  {
    float* oz = a.out_dtype == 0 ? static_cast<float*>(a.out) : a.acc;
    const int64_t ld = a.out_dtype == 0 ? a.ldo : d;
    const int64_t n4 = (int64_t)m * (d / 4);
    for (int64_t i = (int64_t)cta * kHdThreads + tid; i < n4; i += (int64_t)G * kHdThreads) {
      const int64_t r = i / (d / 4), c = (i % (d / 4)) * 4;
      *reinterpret_cast<float4*>(oz + r * ld + c) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t i = (int64_t)cta * kHdThreads + tid; i < t2tot; i += (int64_t)G * kHdThreads) a.t2acc[i] = 0.0f;
    if (cta == 0)
      for (int i = tid; i < kHdCtrl; i += kHdThreads) a.ctrl_next[i] = 0;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(&a.ctrl[0], 1);
    }
  }
  if (dbg != nullptr && tid == 0) dbg[1] = globaltimer();
  const long long Tot = (long long)U * (KT + KT / 2);
  HRange rng;
  rng.init(Tot, G, nT, nV);

  if (warp >= kHdCons) {
    if constexpr (CF::kSetMaxNreg) {  // registers from the producer warpgroup to the consumers
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CF::kProdRegs));
      if (warp >= kHdCons + kHdProd) return;  // the warpgroup's idle warps
    }
    // ---------------- producer warps: both walk every event; producer p streams the stages
    // n with n % kHdProd == p and publishes their descriptors once the next copy event
    // (whoever streams it) shows that no more trailing flags follow.  The walk is plain
    // nested loops over register state (a generator object lived in local memory and
    // cost ~1000 cycles per event).
    const int p = warp - kHdCons;
    const uint64_t pol = policy_evict_first();
    int n = 0, held = -1, xj = -1;
    HDesc hd{};
    bool hwait = false;
    uint16_t tail = 0;
    long long twait = 0;
    HMats X;
    const int UPr = KT + KT / 2, d64 = d / 64, nchT = (KT + kHdTK - 1) / kHdTK;
    const long long lo = rng.lo(cta), hi = rng.lo(cta + 1);
    // The event walk, as one state machine over register scalars with a single
    // emit site (an inlined emit per event kind made the producer ~10K SASS
    // instructions and thrashed the SM sub-partitions' instruction caches).
    // Order: T items | the piece straddling the range end | whole units | the
    // piece straddling the range start | V2 items.
    int ulo = 0, uhi = 0, olo = 0, ohi = 0, npc = 0;
    if (lo < hi) {
      ulo = (int)(lo / UPr);
      uhi = (int)(hi / UPr);
      olo = (int)(lo - (long long)ulo * UPr);
      ohi = (int)(hi - (long long)uhi * UPr);
      npc = ulo == uhi ? 1 : (ohi > 0) + (uhi - ulo - (olo > 0)) + (olo > 0);
    }
    int phase = 0, it = cta, pk = 0, sub = -1, k = 0, mt = 0;
    int pu = 0, po0 = 0, po1 = 0, pj = 0, pc = 0;
    HEv ev;
    // piece pkx of this CTA's range -> (unit, first pair, end pair)
    auto piece_of = [&](int pkx, int& u, int& o0, int& o1) {
      if (ulo == uhi) {
        u = ulo; o0 = olo; o1 = ohi;
        return;
      }
      const int first = ohi > 0, nwhole = uhi - ulo - (olo > 0);
      if (pkx < first) {
        u = uhi; o0 = 0; o1 = ohi;
      } else if (pkx < first + nwhole) {
        u = ulo + (olo > 0) + (pkx - first); o0 = 0; o1 = UPr;
      } else {
        u = ulo; o0 = olo; o1 = UPr;
      }
    };
    // L2 prefetch of piece pkx's weights (W1|W3 columns, W2 rows): the ring's copies then
    // find them in L2 instead of waiting a loaded-HBM round trip (producer 0 only)
    auto prefetch_piece = [&](int pkx) {
      if (p != 0 || pkx >= npc || (a.dbg_flags & 64)) return;
      int u, o0, o1;
      piece_of(pkx, u, o0, o1);
      int j = 0;
      while (j + 1 < np && parts[j + 1].u0 <= u) ++j;
      const HPart& P = parts[j];
      const DecExpert& XE = a.experts[P.e];
      const int c = u - P.u0;
      const int p1a = min(o0, KT), p1b = min(o1, KT);
      const int q0 = max(o0, KT) - KT, q1 = max(o1, KT) - KT;
      if (p1b > p1a && lane < 2)
        prefetch_l2(XE.m[lane].w + ((int64_t)c * KT + p1a) * kTileBytes, (uint32_t)(p1b - p1a) * kTileBytes);
      const uint8_t* w2 = XE.m[2].w;
      for (int S = q0 + lane; S < q1; S += 32) prefetch_l2(w2 + ((int64_t)S * P.kt2 + 2 * c) * kTileBytes, 2 * kTileBytes);
    };
    prefetch_piece(0);
    for (;;) {
      bool have = false;
      if (phase == 0) {  // T items
        if (it < nT) {
          int j = 0;
          while (j + 1 < np && parts[j + 1].tb <= it) ++j;
          const HPart& P = parts[j];
          int l = it - P.tb;
          const int m0 = P.nks[0] * nchT;
          ev.type = EV_T;
          ev.j = j;
          ev.mat = l >= m0;
          if (l >= m0) l -= m0;
          ev.c = l / nchT;
          ev.a = (l % nchT) * kHdTK;
          ev.n = min(kHdTK, KT - ev.a);
          ev.aux = 0;
          it += G;
          have = true;
        } else {
          phase = 1;
        }
      } else if (phase == 1) {  // unit pieces
        if (sub < 0) {
          if (pk >= npc) {
            phase = 2;
            it = G - 1 - cta;
            continue;
          }
          piece_of(pk, pu, po0, po1);
          prefetch_piece(pk + 1);
          pj = 0;
          while (pj + 1 < np && parts[pj + 1].u0 <= pu) ++pj;
          pc = pu - parts[pj].u0;
          sub = 0;
          k = min(po0, KT);
        }
        const HPart& P = parts[pj];
        const int p1a = min(po0, KT), p1b = min(po1, KT);
        const int q0 = max(po0, KT) - KT, q1 = max(po1, KT) - KT;
        ev.j = pj;
        ev.c = pc;
        ev.aux = 0;
        if (sub == 0) {  // P1 stages, then the piece's finish flags
          if (k < p1b) {
            ev.type = EV_P1;
            ev.a = k;
            ev.n = min((int)P.ksp, p1b - k);
            ev.aux = k == p1a;
            ev.mat = 0;
            k += ev.n;
            have = true;
          } else if (p1b == p1a) {  // no P1 part: a P2 tail, h comes from the tail holder
            hwait = true;
            tail = (uint16_t)rng.owner((long long)pu * UPr + KT - 1);
            sub = 3;
            k = 0;
          } else if (p1b < KT) {
            hd.flags |= F_HEADPUB;
            sub = 3;
            k = 0;
          } else {
            hd.flags |= F_FINBEGIN;
            hd.head = (uint16_t)(p1a > 0 ? rng.owner((long long)pu * UPr) : cta);
            sub = 1;
            mt = 0;
            k = 0;
          }
        } else if (sub == 1) {  // FIN-V stages (w1, w3), then SwiGLU
          while (mt < 2 && k >= P.nks[mt]) {
            ++mt;
            k = 0;
          }
          if (mt < 2) {
            ev.type = EV_FV;
            ev.mat = mt;
            ev.a = k;
            ev.n = min(CF::kFV, P.nks[mt] - k);
            k += ev.n;
            have = true;
          } else {
            hd.flags |= F_FINH | (po1 < UPr ? F_PUBH : 0);
            sub = 2;
            k = 0;
          }
        } else if (sub == 2) {  // FIN-U stages (t2 = h U2)
          if (k < P.nks[2]) {
            ev.type = EV_FU;
            ev.a = k;
            ev.n = min(CF::kFU, P.nks[2] - k);
            ev.mat = 0;
            k += ev.n;
            have = true;
          } else {
            if (P.nks[2] > 0) hd.flags |= F_T2DONE;
            sub = 3;
            k = 0;
          }
        } else {  // P2 stages (contiguous slab ranges for the TMA boxes), their order rotated
                  // per CTA so the grid's output reductions do not all hit the same columns at once
          const int nst = (q1 - q0 + CF::kP2 - 1) / CF::kP2;
          if (k < nst) {
            const int kk = (k + cta) % nst;
            ev.type = EV_P2;
            ev.a = q0 + kk * CF::kP2;
            ev.n = min(CF::kP2, q1 - ev.a);
            ev.mat = 0;
            ++k;
            have = true;
          } else {
            sub = -1;
            ++pk;
          }
        }
      } else if (phase == 2) {  // V2 items
        if (it < nV) {
          int j = 0;
          while (j + 1 < np && parts[j + 1].vb <= it) ++j;
          const HPart& P = parts[j];
          const int l = it - P.vb, nks = P.nks[2];
          ev.type = EV_V2;
          ev.j = j;
          ev.a = 0;
          if (nks <= kHdV2K) {
            const int ns = max(1, min(16, kHdStage / (nks * 1024 + 256 * P.gpr[2])));
            ev.c = l * ns;
            ev.n = min(ns, d64 - ev.c);
            ev.aux = 0;
            ev.mat = nks;
          } else {
            const int nsc = (nks + kHdV2K - 1) / kHdV2K;
            ev.c = l / nsc;
            ev.n = 1;
            ev.aux = (l % nsc) * kHdV2K;
            ev.mat = min(kHdV2K, nks - ev.aux);
          }
          it += G;
          have = true;
        } else {
          break;
        }
      }
      if (!have) continue;
      // ---- the single emit site: publish the previous stage if ours, stream this one if ours
      if (held >= 0 && lane == 0) {
        desc[held] = hd;
        mbar_arrive(&full[held]);
      }
      held = -1;
      const int s = n % NS;
      if ((n & (kHdProd - 1)) == p) {
        const HPart& P = parts[ev.j];
        if (ev.j != xj) {
          X.load(a.experts[P.e], a.w2maps + (int64_t)P.e * 128);
          xj = ev.j;
        }
        const uint32_t r = (uint32_t)(n / NS);
        if (r > 0 && !(a.dbg_flags & 16)) {  // experiment bit 4: the producers run alone
          const long long t0 = dbg != nullptr ? clock64() : 0;
          mbar_wait(&empty[s], (r - 1) & 1u);
          if (dbg != nullptr) twait += clock64() - t0;
        }
        const bool nocopy = (a.dbg_flags & 4) != 0;  // experiment: consumers compute on stale stage bytes
        if (lane == 0 && !nocopy) mbar_expect_tx(&full[s], ev_bytes(ev, P));
        __syncwarp();
        const int nc = nocopy ? 0 : ev_ncopies(ev, P);
        for (int i = lane; i < nc; i += 32) {
          const HCopy c = ev_copy(a, X, ev, P, KT, i);
          if (c.tma)
            tma_2d_g2s_hint(ring + s * kHdStage + c.dst, c.src, c.x, c.y, &full[s], pol);
          else
            bulk_g2s_hint(ring + s * kHdStage + c.dst, c.src, c.bytes, &full[s], pol);
        }
        held = s;
        if (dbg != nullptr && lane == 0 && n < 64) a.dbg[(int64_t)kHdDbgG * 128 + (int64_t)cta * 64 + n] = globaltimer();
      }
      hd = HDesc{};
      hd.type = (uint8_t)ev.type;
      hd.j = (uint8_t)ev.j;
      hd.n = (uint8_t)ev.n;
      hd.c = (uint16_t)ev.c;
      hd.a = (uint16_t)ev.a;
      hd.mat = (uint8_t)ev.mat;
      hd.aux = (uint16_t)ev.aux;
      if (ev.type == EV_P1 && ev.aux) hd.flags |= F_FIRST;
      if (hwait) {
        hd.flags |= F_HWAIT;
        hd.tail = tail;
        hwait = false;
      }
      ++n;
    }
    // the last stage's descriptor, then an END descriptor in a stage of its own
    if (held >= 0 && lane == 0) {
      desc[held] = hd;
      mbar_arrive(&full[held]);
    }
    if ((n & (kHdProd - 1)) == p && !(a.dbg_flags & 16)) {
      const int s = n % NS;
      if (n >= NS) mbar_wait(&empty[s], ((uint32_t)(n / NS) - 1) & 1u);
      if (lane == 0) {
        HDesc e{};
        e.flags = F_END;
        desc[s] = e;
        mbar_arrive(&full[s]);
      }
    }
    if (dbg != nullptr && lane == 0 && p == 0) {
      dbg[3] = globaltimer();
      dbg[126] = twait;
    }
    return;
  }

  // ---------------- consumer warps
  if constexpr (CF::kSetMaxNreg) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CF::kConsRegs));
  if (a.dbg_flags & 16) return;
  DqConsts* dqs = reinterpret_cast<DqConsts*>(smem + CF::kOffDq);
  if (tid < 2) dqs[tid] = make_dq_consts(tid);
  cons_bar<NT>();
  float accP[2][4][NT][4];
  const int ct = tid;  // consumer thread 0 .. kCT - 1
  int n = 0, nev = 0;
  long long cwait = 0;
  bool zero_seen = false;
  int tc_tag = -1;  // participant whose t (ranks <= 64) is in tcache
  const int nch = (KT + kHdTK - 1) / kHdTK;
  int slot = 0;
  uint32_t fph = 0;  // full-barrier phase parity of `slot`
  for (;;) {
    {
      const long long t0 = dbg != nullptr ? clock64() : 0;
      const long long g0 = dbg != nullptr && tid == 0 ? globaltimer() : 0;
      mbar_wait(&full[slot], fph);
      if (dbg != nullptr) cwait += clock64() - t0;
      if (dbg != nullptr && tid == 0 && n < 64) {
        long long* w = a.dbg + (int64_t)kHdDbgG * 192 + ((int64_t)cta * 64 + n) * 2;
        w[0] = g0;
        w[1] = globaltimer();
      }
    }
    ++n;
    const HDesc D = desc[slot];
    const uint8_t* st = ring + slot * kHdStage;
    if (__builtin_expect(D.flags & F_HWAIT, 0)) {  // h of this unit from its tail holder
      cons_bar<NT>();  // hbuf may still be read by the previous piece's P2 events
      for (int w = ct; w < 8 * NT * 32; w += kCT) {
        const int tok = w >> 5, wi = w & 31;
        const uint32_t hv = wait_tagged(a.hpub + ((int64_t)D.tail * 16 + tok) * 32 + wi, a.epoch);
        *reinterpret_cast<uint32_t*>(hbuf + tok * 72 + 2 * wi) = hv;
      }
      cons_bar<NT>();
    }

    // ---- hot path: a P1 stage with no trailing steps (kept compact and in line; the
    // consumer's per-stage overhead is instruction-fetch bound when it branches around)
    if (__builtin_expect(D.type == EV_P1 && (D.flags & ~F_FIRST) == 0, 1)) {
      const HPart& P = parts[D.j];
      const DqConsts dq = dqs[P.mode & 1];
      if (D.flags & F_FIRST) {
#pragma unroll
        for (int x = 0; x < kAcc; ++x) accel<NT>(accP, x) = 0.0f;
      }
      const __half* xs = reinterpret_cast<const __half*>(st + 2 * D.n * kTileBytes);
      const int xrs = D.n * 32 + 8;
      const int l_end = (a.dbg_flags & 32) ? 0 : D.n;  // experiment bit 5: no P1 compute
#pragma unroll 1
      for (int l = warp; l < l_end; l += kHdCons) {
        BTile<NT> b;
        load_bs<NT>(b, xs, xrs, P.rows, l * 32, g, q);
        tile_real<NT, 2, 2>(st + l * kTileBytes, D.n * kTileBytes, b, accP, dq, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == NS) {
        slot = 0;
        fph ^= 1u;
      }
      if (dbg != nullptr && tid == 0 && nev < 60) {
        dbg[4 + 2 * nev] = D.type | (D.n << 8) | ((long long)D.flags << 16) | ((long long)D.j << 32);
        dbg[5 + 2 * nev] = globaltimer();
        ++nev;
      }
      continue;
    }
    // ---- hot path: a P2 stage (out += wt * h_c W2[c rows, d-slabs]; slab pairs (l, l + kCons))
    if (__builtin_expect(D.type == EV_P2 && (D.flags & ~F_HWAIT) == 0, 1)) {
      const HPart& P = parts[D.j];
      const DqConsts dq = dqs[P.mode & 1];
      if (!zero_seen) {
        wait_count(a.ctrl, G);
        zero_seen = true;
      }
      BTile<NT> b0, b1;
      load_bs<NT>(b0, hbuf, 72, 16, 0, g, q);
      load_bs<NT>(b1, hbuf, 72, 16, 32, g, q);
      // warp w: slab pairs (w + 2 kCons p, w + 2 kCons p + kCons), p = 0 .. kP2 / (2 kCons) - 1
      constexpr int L2 = kHdCons;
      float acc2[2][4][NT][4];
      const int p2_end = (a.dbg_flags & 128) ? 0 : D.n;  // experiment bit 7: no P2 compute
#pragma unroll 1
      for (int l = warp; l < p2_end; l += 2 * kHdCons) {
        const bool two = l + L2 < D.n;
#pragma unroll
        for (int x = 0; x < kAcc; ++x) accel<NT>(acc2, x) = 0.0f;
        tile_real<NT, 2, 2>(st + l * 2 * kTileBytes, two ? L2 * 2 * kTileBytes : 0, b0, acc2, dq, lane);
        tile_real<NT, 2, 2>(st + l * 2 * kTileBytes + kTileBytes, two ? L2 * 2 * kTileBytes : 0, b1, acc2, dq, lane);
        if (!(a.dbg_flags & 2)) {
          hd_epi_slab<NT>(a, P, acc2[0], D.a + l, lane);
          if (two) hd_epi_slab<NT>(a, P, acc2[1], D.a + l + L2, lane);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == NS) {
        slot = 0;
        fph ^= 1u;
      }
      if (dbg != nullptr && tid == 0 && nev < 60) {
        dbg[4 + 2 * nev] = D.type | (D.n << 8) | ((long long)D.flags << 16) | ((long long)D.j << 32);
        dbg[5 + 2 * nev] = globaltimer();
        ++nev;
      }
      continue;
    }
    if (D.flags & F_END) break;
    const HPart& P = parts[D.j];
    const DqConsts dq = dqs[P.mode & 1];
    const int rows = P.rows;

    switch (D.type) {
      case EV_T: {  // t partial of (j, mat, rank group c) over k-tiles [a, a + n)
        const __half* xs = reinterpret_cast<const __half*>(st + D.n * kPseudoInt3Bytes);
        const int xrs = D.n * 32 + 8;
        float accT[1][4][NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) accT[0][0][nt][e] = 0.0f;
        for (int l = warp; l < D.n; l += kHdCons) {
          BTile<NT> b;
          load_bs<NT>(b, xs, xrs, rows, l * 32, g, q);
          tile_pseudo<NT, 1>(st + l * kPseudoInt3Bytes, false, b, accT, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) red[((warp * NT + nt) * 4 + e) * 32 + lane] = accT[0][0][nt][e];
        cons_bar<NT>();
        if (warp == 0) {
          const int t = P.tb + D.mat * P.nks[0] * nch + D.c * nch + D.a / kHdTK;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float s = 0.0f;
#pragma unroll
              for (int w = 0; w < kHdCons; ++w) s += red[((w * NT + nt) * 4 + e) * 32 + lane];
              const int tok = 8 * nt + 2 * q + (e & 1), rk = g + 8 * (e >> 1);
              st_tagged1(a.tpart + ((int64_t)t * 16 + tok) * 16 + rk, s, a.epoch);
            }
        }
        cons_bar<NT>();
        break;
      }
      case EV_P1: {
        if (D.flags & F_FIRST) {
#pragma unroll
          for (int x = 0; x < kAcc; ++x) accel<NT>(accP, x) = 0.0f;
        }
        const __half* xs = reinterpret_cast<const __half*>(st + 2 * D.n * kTileBytes);
        const int xrs = D.n * 32 + 8;
#pragma unroll 1
        for (int l = warp; l < D.n; l += kHdCons) {
          BTile<NT> b;
          load_bs<NT>(b, xs, xrs, rows, l * 32, g, q);
          tile_real<NT, 2, 2>(st + l * kTileBytes, D.n * kTileBytes, b, accP, dq, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        break;
      }
      case EV_FV: {  // ybuf[mat] += (t V) of slab c, rank steps [a, a + n)
        // t of these rank steps, summed over the T items' k chunks (fixed order): ranks <= 64
        // from the per-participant cache (loaded once for both matrices), else staged in red
        const bool small = P.nks[0] <= 4 && P.nks[1] <= 4;
        float* tsrc = red;
        int trs = 16 * D.n + 8, tcol = 0;
        if (small) {
          tsrc = tcache + D.mat * 8 * NT * 72;
          trs = 72;
          tcol = 16 * D.a;
        }
        if (!small || tc_tag != D.j) {
          const int nmat = small ? 2 : 1;
          const int w_per = 8 * NT * (small ? 64 : 16 * D.n);
          for (int w = ct; w < nmat * w_per; w += kCT) {
            const int mt = small ? w / w_per : D.mat, w2 = w % w_per;
            const int cols = small ? 64 : 16 * D.n;
            const int tok = w2 / cols, rr = w2 % cols;
            const int ks = (small ? 0 : D.a) + (rr >> 4);
            float s = 0.0f;
            if (ks < P.nks[mt]) {
              const int tbase = P.tb + mt * P.nks[0] * nch;
              const uint64_t* tp = a.tpart + ((int64_t)(tbase + ks * nch) * 16 + tok) * 16 + (rr & 15);
              for (int c0 = 0; c0 < nch; c0 += 8) {  // 8 loads in flight, then the tag checks
                uint64_t wv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) wv[u] = c0 + u < nch ? ld_relaxed_b64(tp + (int64_t)(c0 + u) * 256) : 0ull;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                  if (c0 + u < nch) {
                    if ((uint32_t)(wv[u] >> 32) != (uint32_t)a.epoch)
                      wv[u] = wait_tagged(tp + (int64_t)(c0 + u) * 256, a.epoch);
                    s += __uint_as_float((uint32_t)wv[u]);
                  }
              }
            }
            if (small)
              tcache[(mt * 8 * NT + tok) * 72 + rr] = s;
            else
              red[tok * trs + rr] = s;
          }
          if (small) tc_tag = D.j;
          cons_bar<NT>();
        }
        constexpr int kHalves = kHdCons / 4;
        const int i = warp & 3, half = warp >> 2;
        const int gpr = P.gpr[D.mat];
        const float* vst = reinterpret_cast<const float*>(st + D.n * kVftInt3Bytes);
        float accY[NT][4], Dm[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) accY[nt][e] = Dm[nt][e] = 0.0f;
        int gcur = -1;
        for (int l = half; l < D.n; l += kHalves) {
          const int gr = (D.a + l) >> 2;
          if (gr != gcur) {
            if (gcur >= 0) {
              const float s0 = vst[(16 * i + g) * gpr + gcur], s1 = vst[(16 * i + g + 8) * gpr + gcur];
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                accY[nt][0] += s0 * Dm[nt][0];
                accY[nt][1] += s0 * Dm[nt][1];
                accY[nt][2] += s1 * Dm[nt][2];
                accY[nt][3] += s1 * Dm[nt][3];
                Dm[nt][0] = Dm[nt][1] = Dm[nt][2] = Dm[nt][3] = 0.0f;
              }
            }
            gcur = gr;
          }
          const uint2 cw = *reinterpret_cast<const uint2*>(st + l * kVftInt3Bytes + lane * 32 + i * 8);
          const uint32_t A[4] = {codes_h2(cw.x, false), codes_h2(cw.x, true), codes_h2(cw.y, false),
                                 codes_h2(cw.y, true)};
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const float* tr = tsrc + (8 * nt + g) * trs + tcol + 16 * l + 2 * q;
            const float2 t0 = *reinterpret_cast<const float2*>(tr), t1 = *reinterpret_cast<const float2*>(tr + 8);
            uint32_t bh0, bl0, bh1, bl1;
            split_h2(t0.x, t0.y, bh0, bl0);
            split_h2(t1.x, t1.y, bh1, bl1);
            mma_16816(Dm[nt], A, bh0, bh1);
            mma_16816(Dm[nt], A, bl0, bl1);
          }
        }
        if (gcur >= 0) {
          const float s0 = vst[(16 * i + g) * gpr + gcur], s1 = vst[(16 * i + g + 8) * gpr + gcur];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            accY[nt][0] += s0 * Dm[nt][0];
            accY[nt][1] += s0 * Dm[nt][1];
            accY[nt][2] += s1 * Dm[nt][2];
            accY[nt][3] += s1 * Dm[nt][3];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
#pragma unroll
        for (int hh = 0; hh < kHalves; ++hh) {
          if (half == hh)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e) ybuf[(((D.mat * 4 + i) * NT + nt) * 4 + e) * 32 + lane] += accY[nt][e];
          cons_bar<NT>();
        }
        break;
      }
      case EV_FU: {  // t2 += h_c U2[c rows], rank groups [a, a + n)
        if (!zero_seen) {
          wait_count(a.ctrl, G);
          zero_seen = true;
        }
        BTile<NT> b0, b1;
        load_bs<NT>(b0, hbuf, 72, 16, 0, g, q);
        load_bs<NT>(b1, hbuf, 72, 16, 32, g, q);
        const int r16 = 16 * P.nks[2];
        for (int l = warp; l < D.n; l += kHdCons) {
          float accU[1][4][NT][4];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) accU[0][0][nt][e] = 0.0f;
          tile_pseudo<NT, 1>(st + l * 2 * kPseudoInt3Bytes, false, b0, accU, lane);
          tile_pseudo<NT, 1>(st + l * 2 * kPseudoInt3Bytes + kPseudoInt3Bytes, false, b1, accU, lane);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int tok = 8 * nt + 2 * q + (e & 1), rk = 16 * (D.a + l) + g + 8 * (e >> 1);
              if (tok < rows) red_add_f32(a.t2acc + P.t2off + tok * r16 + rk, accU[0][0][nt][e]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        break;
      }
      case EV_V2: {  // out += wt * (t2 V2) of d-slabs [c, c + n), rank steps [aux, aux + mat)
        if (!zero_seen) {
          wait_count(a.ctrl, G);
          zero_seen = true;
        }
        if (lane == 0) wait_count(a.ctrl + 4 + D.j, P.nu);
        __syncwarp();
        const int nk = D.mat, gpr = P.gpr[2], r16 = 16 * P.nks[2];
        // t2 of these rank steps -> [8 NT][16 nk + 8] behind the epilogue scratch (zero rows past `rows`)
        float* tsm = red + CF::kScrBytes / 4;
        const int trs = 16 * nk + 8;
        cons_bar<NT>();  // every warp is past the previous V2 item's reads of tsm
        for (int w = ct; w < 8 * NT * 16 * nk; w += kCT) {
          const int tok = w / (16 * nk), rr = w % (16 * nk);
          tsm[tok * trs + rr] = tok < rows ? __ldcg(a.t2acc + P.t2off + tok * r16 + 16 * D.aux + rr) : 0.0f;
        }
        cons_bar<NT>();
        const float* vst = reinterpret_cast<const float*>(st + D.n * nk * kVftInt3Bytes);
          for (int l = warp; l < D.n; l += kHdCons) {
          float acc[4][NT][4], Dm[4][NT][4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[i][nt][e] = Dm[i][nt][e] = 0.0f;
          int gcur = -1;
          for (int kk = 0; kk < nk; ++kk) {
            const int gr = (D.aux + kk) >> 2;
            if (gr != gcur) {
              if (gcur >= 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float s0 = vst[(l * 64 + 16 * i + g) * gpr + gcur];
                  const float s1 = vst[(l * 64 + 16 * i + g + 8) * gpr + gcur];
#pragma unroll
                  for (int nt = 0; nt < NT; ++nt) {
                    acc[i][nt][0] += s0 * Dm[i][nt][0];
                    acc[i][nt][1] += s0 * Dm[i][nt][1];
                    acc[i][nt][2] += s1 * Dm[i][nt][2];
                    acc[i][nt][3] += s1 * Dm[i][nt][3];
                    Dm[i][nt][0] = Dm[i][nt][1] = Dm[i][nt][2] = Dm[i][nt][3] = 0.0f;
                  }
                }
              }
              gcur = gr;
            }
            uint32_t bh[NT][2], bl[NT][2];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const float* tr = tsm + (8 * nt + g) * trs + 16 * kk + 2 * q;
              const float2 v0 = *reinterpret_cast<const float2*>(tr), v1 = *reinterpret_cast<const float2*>(tr + 8);
              split_h2(v0.x, v0.y, bh[nt][0], bl[nt][0]);
              split_h2(v1.x, v1.y, bh[nt][1], bl[nt][1]);
            }
            const uint4* src = reinterpret_cast<const uint4*>(st + (l * nk + kk) * kVftInt3Bytes + lane * 32);
            const uint4 c0 = src[0], c1 = src[1];
            const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t A[4] = {codes_h2(cw[2 * i], false), codes_h2(cw[2 * i], true),
                                     codes_h2(cw[2 * i + 1], false), codes_h2(cw[2 * i + 1], true)};
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                mma_16816(Dm[i][nt], A, bh[nt][0], bh[nt][1]);
                mma_16816(Dm[i][nt], A, bl[nt][0], bl[nt][1]);
              }
            }
          }
          if (gcur >= 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float s0 = vst[(l * 64 + 16 * i + g) * gpr + gcur];
              const float s1 = vst[(l * 64 + 16 * i + g + 8) * gpr + gcur];
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                acc[i][nt][0] += s0 * Dm[i][nt][0];
                acc[i][nt][1] += s0 * Dm[i][nt][1];
                acc[i][nt][2] += s1 * Dm[i][nt][2];
                acc[i][nt][3] += s1 * Dm[i][nt][3];
              }
            }
          }
          hd_epi_slab<NT>(a, P, acc, D.c + l, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        break;
      }
      default: break;
    }

    // ---- trailing steps of this stage
    if (D.flags & (F_HEADPUB | F_FINBEGIN)) {
      // reduction of accP over the consumer warps into warp 0, in a fixed order through
      // at most 4 warp slots of red: fold the top 4 warps onto the 4 below them while
      // more than 8 remain, then halve
      cons_bar<NT>();
#pragma unroll 1
      for (int cnt = kHdCons; cnt > 1;) {
        const int k = cnt > 8 ? 4 : cnt / 2;  // writers [cnt - k, cnt) -> readers [cnt - 2k, cnt - k)
        if (warp >= cnt - k && warp < cnt)
#pragma unroll
          for (int x = 0; x < kAcc; ++x) red[((warp - (cnt - k)) * kAcc + x) * 32 + lane] = accel<NT>(accP, x);
        cons_bar<NT>();
        if (warp >= cnt - 2 * k && warp < cnt - k)
#pragma unroll
          for (int x = 0; x < kAcc; ++x) accel<NT>(accP, x) += red[((warp - (cnt - 2 * k)) * kAcc + x) * 32 + lane];
        cons_bar<NT>();
        cnt -= k;
      }
      if (warp == 0) {
        if (D.flags & F_HEADPUB) {
#pragma unroll
          for (int x = 0; x < kAcc; ++x)
            st_tagged1(a.part + (int64_t)cta * 1024 * NT + x * 32 + lane, accel<NT>(accP, x), a.epoch);
        } else {
          float hs[kAcc];
#pragma unroll
          for (int x = 0; x < kAcc; ++x) hs[x] = 0.0f;
          for (int c2 = D.head; c2 < cta; ++c2) {
            if (rng.lo(c2) == rng.lo(c2 + 1)) continue;  // empty range
            const uint64_t* pp = a.part + (int64_t)c2 * 1024 * NT + lane;
            uint64_t wv[kAcc];
#pragma unroll
            for (int x = 0; x < kAcc; ++x) wv[x] = ld_relaxed_b64(pp + x * 32);  // all in flight
#pragma unroll
            for (int x = 0; x < kAcc; ++x) {
              if ((uint32_t)(wv[x] >> 32) != (uint32_t)a.epoch) wv[x] = wait_tagged(pp + x * 32, a.epoch);
              hs[x] += __uint_as_float((uint32_t)wv[x]);
            }
          }
          // ybuf element ((mat * 4 + i) * NT + nt) * 4 + e) * 32 + lane == x * 32 + lane
#pragma unroll
          for (int x = 0; x < kAcc; ++x) ybuf[x * 32 + lane] = hs[x] + accel<NT>(accP, x);
        }
      }
      cons_bar<NT>();
    }
    if (D.flags & F_FINH) {  // SwiGLU -> h (binary16) in hbuf; publish when a P2 tail is elsewhere
      for (int el = ct; el < 512 * NT; el += kCT) {
        const int ln = el & 31, e = (el >> 5) & 3, nt = (el >> 7) % NT, i = (el >> 7) / NT;
        const int tok = 8 * nt + 2 * (ln & 3) + (e & 1), nn = 16 * i + (ln >> 2) + 8 * (e >> 1);
        const float y1 = ybuf[el], y3 = ybuf[512 * NT + el];
        float h = __fdividef(y1, 1.0f + __expf(-y1)) * y3;
        if (tok >= rows) h = 0.0f;
        hbuf[tok * 72 + nn] = __float2half_rn(h);
      }
      cons_bar<NT>();
      if (D.flags & F_PUBH) {
        for (int w = ct; w < 8 * NT * 32; w += kCT) {
          const int tok = w >> 5, wi = w & 31;
          const uint32_t hv = *reinterpret_cast<const uint32_t*>(hbuf + tok * 72 + 2 * wi);
          const uint64_t word = ((uint64_t)(uint32_t)a.epoch << 32) | hv;
          asm volatile("st.global.cg.b64 [%0], %1;" ::"l"(a.hpub + ((int64_t)cta * 16 + tok) * 32 + wi), "l"(word)
                       : "memory");
        }
      }
    }
    if (D.flags & F_T2DONE) {  // the unit's t2 reductions (all consumer warps) -> the expert's counter
      cons_bar<NT>();
      if (ct == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.ctrl + 4 + D.j) : "memory");
    }
    if (dbg != nullptr && tid == 0 && nev < 60) {
      dbg[4 + 2 * nev] = D.type | (D.n << 8) | ((long long)D.flags << 16) | ((long long)D.j << 32);
      dbg[5 + 2 * nev] = globaltimer();
      ++nev;
    }
    if (++slot == NS) {
      slot = 0;
      fph ^= 1u;
    }
  }
  if (dbg != nullptr && tid == 0) {
    dbg[2] = globaltimer();
    dbg[127] = cwait;
    dbg[125] = nev;
  }
  // f16 output: the last CTA to finish converts the fp32 accumulator
  if (a.out_dtype != 0) {
    cons_bar<NT>();
    if (ct == 0) {
      __threadfence();
      misc[8] = atomicAdd(&a.ctrl[1], 1) == G - 1;
      __threadfence();
    }
    cons_bar<NT>();
    if (misc[8]) {
      for (int64_t i = ct; i < (int64_t)m * d; i += kCT) {
        const int64_t r = i / d, c = i % d;
        static_cast<__half*>(a.out)[r * a.ldo + c] = __float2half_rn(__ldcg(a.acc + i));
      }
    }
  }
}

}  // namespace milo_dev
