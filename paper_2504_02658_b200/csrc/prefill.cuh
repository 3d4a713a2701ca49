// K3: the prefill-regime W3A16 + LoRC GEMM on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM), for token counts where the weights are
// worth reusing across many tokens (m_e >= ~64 per matrix).
//
// Reference semantics, per matrix: milo::gemm_w3a16 (proj/src/gemm.cpp:117-199)
//   C = half(A) * dequant(W) + (half(A) U) V, fp32 accumulation.
//
// Per work item (problem p, n-tile of 128 output columns = 2 slabs, token tile
// of <= 128 rows) one CTA computes D[128 n][ntok] = W^T X^T in TMEM:
//   * packed producer : cp.async.bulk of the packed INT3 macro tiles, one run of
//                       4 k-tiles per (matrix, slab) per 128-k ring slot;
//   * image producer  : the activation images (binary16, SW128 K-major, built by
//                       pf_image_kernel / pf_img_t_kernel) of a stage pair in one
//                       copy, and the LoRC t images;
//   * dequant groups  : packed tiles -> bit-exact binary16 W^T written into TMEM
//                       (tcgen05.st from each warp's lane quarter), the A operand;
//   * ring waiter     : waits on the A / B rings, publishes a stage counter;
//   * two MMA issuers : tcgen05.mma.kind::f16 with A from TMEM (K = 16, 4 per
//                       matrix per 64-k stage), tcgen05.commit releases the slots;
//   * epilogue warps  : tcgen05.ld (32 lanes x 16 columns) -> C rows / SwiGLU.
// The compensator term (t V) runs as extra K stages of the same accumulator:
// A = V^T image rows (hi or lo binary16 half of the fp32 values, copied into the
// TMEM slot), B = t image (hi or lo), three MMAs per 64-rank chunk (hi.hi +
// hi.lo + lo.hi), i.e. fp32-level accuracy on the tensor cores.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "layout.cuh"
#include "ptx.cuh"

namespace milo_dev {

#ifndef PF_GROUPS
#define PF_GROUPS 2  // dequant groups (4 warps each; 2 measured faster than 3 or 4: 96 registers at 17 warps)
#endif
#ifndef PF_PS2
#define PF_PS2 5  // packed ring slots (128 k each) of the two-matrix / two-n-tile variants
#endif
#ifndef PF_PROF
#define PF_PROF 0  // experiments: per-role cycle split of CTA 0 (tools/pf_stage_trace.py)
#endif
#ifndef PF_ISSUERS
#define PF_ISSUERS 2  // MMA-issuing threads (experiments: 1)
#endif
#ifndef PF_VPREFETCH
#define PF_VPREFETCH 0  // 1: packed producer prefetches the item's V^T images to L2 at item start
#endif
#ifndef PF_DQ_ROLLED
#define PF_DQ_ROLLED 1  // the dequant warps' two 64-k halves per stage run one loop body (0: unrolled)
#endif
#ifndef PF_ISSUE_ROLLED
#define PF_ISSUE_ROLLED 0  // 1: the issuers' accumulator loop is not unrolled (smaller kernel)
#endif
#ifndef PF_LMERGE_MIN
// token tiles >= this run one merged LoRC stage per chunk (else 3).  Off by default:
// merged (32) measured DeepSeek batch 256 -30 us but Arctic +300 us, and with it
// compiled out the kernel is ~5% fewer instructions, which alone took Arctic phase 2
// 906 -> 822 us (the roles' loops share the SM's instruction cache; K3)
#define PF_LMERGE_MIN (1 << 20)
#endif
#ifndef PF_MIN_AS
#define PF_MIN_AS 3  // A slots below which the accumulators are single-buffered
#endif
#ifndef PF_B_KB
#define PF_B_KB 128  // activation / t image ring (KB)
#endif
constexpr int kPfM = 128;              // output columns per tile (UMMA M)
constexpr int kPfN = 128;              // tokens per tile (UMMA N, TMEM columns)
constexpr int kPfK = 64;               // k per stage (128 B of binary16 per operand row)
constexpr int kPfImg = kPfN * kPfK * 2;  // 16 KB: one operand image (128 rows x 128 B)
constexpr int kPfPackedPerMat = 2 * 2 * kTileBytes;  // 2 slabs x 2 k-tiles = 3584 B
constexpr int kPfGroupWarps = 4;       // warps per dequant group = the 4 TMEM lane quarters
#ifndef PF_EPI_HALVES
#define PF_EPI_HALVES 2  // epilogue warps per TMEM lane quarter (the second four follow the dequant groups)
#endif
constexpr int kPfEpiWarps = 4 * PF_EPI_HALVES;  // warps 0..3 (+ the last 4): TMEM lanes 32 (w % 4) ..
constexpr int kPfProdWarp = 4;         // packed-weight producer
constexpr int kPfMmaWarp = 5;
constexpr int kPfBWarp = 6;            // activation / t image producer
constexpr int kPfMmaWarp2 = 7;          // second MMA issuer (one thread issues <= 1 MMA per ~55 cycles)
constexpr int kPfWaitWarp = 8;          // waits on the A / B rings for the issuers
constexpr int kPfDeqWarp0 = 9;
constexpr int kPfTraceStages = 256;    // debug timeline: CTA 0's first stages (PfArgs::dbg)
constexpr int kPfDbgLongs = 148 * 8 + kPfTraceStages * 8;  // dbg region of one launch
// NG = n-tiles (128 output columns each) per work item: the item's activation
// image of a stage feeds NG MMAs (NG accumulators), so activation traffic per
// FLOP drops by NG.
// Groups <= A slots: a group that starts stage st has only seen stage
// st - groups consumed, and its parity wait on the slot is unambiguous only
// if the slot's barrier is at most one phase behind (st - 2 AS consumed).
template <int NMAT, int NG = 1>
struct PfRoles {
  static constexpr int kGroups = PF_GROUPS;  // stages de-quantized concurrently
  static constexpr int kDeqWarps = kGroups * kPfGroupWarps;
  static constexpr int kThreads = 32 * (kPfDeqWarp0 + kDeqWarps + 4 * (PF_EPI_HALVES - 1));
};

// The de-quantized weights (the MMA's A operand, W^T) live in TENSOR memory:
// TMEM columns 256..511 hold kAS stages of NG x NMAT 128-row x 64-k binary16
// tiles (32 columns each), written by the dequant warps with tcgen05.st and
// read by tcgen05.mma straight from TMEM -- no shared-memory round trip for
// the weights (the smem-A design moved 32 KB st.shared + 32 KB MMA reads per
// two-matrix stage through the 128 B/clk shared-memory port, its bound at
// small token tiles).  Columns 0..255 hold the fp32 accumulators (double
// buffered when NG x NMAT x ntok fits 128 columns).  Shared memory keeps the
// packed-weight ring and the activation / t image ring.
template <int NMAT, int NG = 1>
struct PfCfg {
  static constexpr int kPS = (NG == 2 || NMAT == 2) ? PF_PS2 : 10;  // packed-weight ring (HBM latency)
  static constexpr int kStageCols = NG * NMAT * 64;  // TMEM columns of one A stage (128 k)
  static constexpr int kASMax = 384 / kStageCols;    // A slots in TMEM (the accumulators take >= 128 columns)
  static constexpr int kBRegion = PF_B_KB * 1024;
  static constexpr int kBSMax = 16;                      // B slots = region / (ntok_max x 128), <= 16
  // the producers move 128 k per ring slot (two 64-k stages): a bulk copy costs
  // its issuing thread ~400-650 cycles whatever its size, so fewer, larger copies
  static constexpr int kStageP = 2 * NG * NMAT * kPfPackedPerMat;  // [nm][slab][4 k-tiles]
  static constexpr int kOffB = 0;                        // 1024-aligned images first
  static constexpr int kOffP = kOffB + kBRegion;
  static constexpr int kOffBar = kOffP + kPS * kStageP;
  // p_full[PS] p_empty[PS] a_full[AS] a_empty[AS] b_full[BSMax] b_empty[BSMax] acc_full[2] acc_empty[2]
  // (B slots: two 64-k activation images of a main-stage pair, or one t image)
  static constexpr int kNumBars = 2 * kPS + 2 * kASMax + 2 * kBSMax + 4;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kOffStage = (kOffTmem + 16 + 127) & ~127;  // epilogue transpose [4 warps][32][33] f32
  static constexpr int kBytes = kOffStage + kPfEpiWarps * 16 * 33 * 4 + 1024;  // + alignment slack
  static constexpr int kTmemCols = 512;
};

// One GEMM problem: a weight matrix (or w1|w3 pair) times a block of token rows.
struct PfProblem {
  const uint8_t* w[2];      // macro tiles (slab-major) of matrix 0 / 1
  const uint8_t* act;       // activation images [tok_tiles][k/64][16 KB]
  const uint8_t* vimg[2];   // V^T images [n/128][r64 chunks][hi, lo][16 KB] (null: no LoRC)
  const uint8_t* timg[2];   // t images  [tok_tiles][r64 chunks][hi, lo][16 KB]
  int32_t rchunks[2];       // 64-rank chunks of each compensator (0: none)
  int32_t k, n, rows;       // rows = tokens of this problem
  int32_t ntok;             // token tile (UMMA N): multiple of 16, <= 128; images are ntok x 128 B
  int32_t mode;
  int32_t kind;             // 0: store rows (f32 / f16), 1: SwiGLU -> binary16 rows
  int32_t out_dtype;
  int64_t ldo;
  void* out;                // row r of the problem -> out + row_map[r] * ldo
  const int32_t* row_map;   // null: identity
};

struct PfArgs {
  int32_t ntok_max;           // largest token tile of the launch: B ring slot = ntok_max x 128 B
  long long* dbg;             // optional per-CTA role timeline (globaltimer ns), [cta][8]
  int32_t flags;              // debug: bit 0 skip dequant math, bit 1 skip MMAs
  const PfProblem* problems;
  int32_t n_problems;
  const int32_t* item_start;  // exclusive prefix of work items per problem (n_problems + 1)
  int32_t n_items;
  // device-planned launches (moe_plan_kernel): n_problems / n_items / ntok_max are
  // read from dev_counts[0..2] at kernel start (null: the host values above)
  const int32_t* dev_counts;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint64_t pf_desc_sw128(uint32_t saddr) {
  // UMMA shared-memory descriptor, K-major SWIZZLE_128B: rows of 128 B, 8-row
  // atoms 1024 B apart (SBO = 64 x 16 B), LBO = 1, version 1 (sm_100).
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)64u << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// Instruction descriptor: kind::f16, A/B binary16 K-major, D fp32, M = 128, N = ntok.
__device__ __forceinline__ uint32_t pf_idesc(int ntok) {
  return (1u << 4) | ((uint32_t)(ntok >> 3) << 17) | ((uint32_t)(kPfM >> 4) << 24);
}
__device__ __forceinline__ void pf_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
// A operand from tensor memory (rows = TMEM lanes, k pairs = columns).
__device__ __forceinline__ void pf_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(accum));
}
// Warp-converged forms: the whole warp executes them, one elected lane issues
// (operands stay in uniform registers -- a lone-lane issuer pays register ->
// uniform moves and an election loop per MMA).
__device__ __forceinline__ void pf_mma_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void pf_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 st;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// 16 lanes x 32 columns: thread (g = lane / 4, q = lane % 4) writes lane g
// (v[4c], v[4c + 1]) and lane g + 8 (v[4c + 2], v[4c + 3]) at columns
// 8c + 2q, 8c + 2q + 1 (c = 0..3) -- the mma.m16n8k16 A-fragment geometry.
__device__ __forceinline__ void tmem_st16x256_x4(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// 32 lanes x 32 columns: thread t writes lane t, columns 0..31 = v[0..31].
__device__ __forceinline__ void tmem_st32x32_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta_shared(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void pf_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// fast SiLU: the result is rounded to binary16 (h rows) right after
__device__ __forceinline__ float pf_silu(float a) { return __fdividef(a, 1.0f + __expf(-a)); }
// Latency-critical handoffs spin on the non-blocking test (no suspend window).
__device__ __forceinline__ void pf_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// Work item -> (problem, n-tile, token tile).  Items of a problem are n-tile
// major so consecutive items share the activation images (L2 reuse).
template <int NG>
__device__ __forceinline__ void pf_item(const PfArgs& a, int item, int& p, int& nt, int& tt) {
  int lo = 0, hi = a.n_problems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.item_start[mid] <= item) lo = mid; else hi = mid - 1;
  }
  p = lo;
  const PfProblem P = a.problems[p];  // by value: fields live in registers
  const int tts = (P.rows + P.ntok - 1) / P.ntok;
  const int rel = item - a.item_start[p];
  nt = rel / tts;
  tt = rel - nt * tts;
}

// One main stage of one dequant warp: for each of the stage's NM matrices /
// n-tiles, the half IH of the 4 units of slab tiles (kt = 0, 1) -> binary16
// W^T rows of TMEM lanes taddr .. + 31 (16x256b stores, n subtiles 2 IH, 2 IH + 1).
template <int IH, int NM>
__device__ __forceinline__ void pf_dequant_stage(const uint8_t* sP, int lane, const DqConsts& dq, uint32_t taddr) {
  const int q = lane & 3;
#pragma unroll
  for (int nm = 0; nm < NM; ++nm) {  // tiles of (nm, slab, kt) at ((nm * 2 + slab) * 2 + kt) * 896
    uint32_t v0[16], v1[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // unit (kt, j) = 16-k block u of the stage
      const int kt = u >> 1, j = u & 1;
      const uint8_t* tile = sP + (nm * 8 + kt) * kTileBytes;  // [nm][slab][4 k-tiles]
      const uint2 wa = *reinterpret_cast<const uint2*>(tile + kPlaneAOff + lane * 16 + 8 * j);
      const uint32_t wb = *reinterpret_cast<const uint32_t*>(tile + kPlaneBOff + lane * 8 + 4 * j);
      const uint4 mm = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32 + 16 * j);
      const uint32_t S2[2] = {mm.x, mm.z}, O2[2] = {mm.y, mm.w};
      uint32_t o[8];
      half_unit_dequant<IH>(wa.x, wa.y, wb, S2, O2, dq, o);
      // o[4 il + r]: row g + 8 (r & 1), k pair q + 4 (r >> 1)
      v0[4 * u + 0] = o[0];
      v0[4 * u + 1] = o[2];
      v0[4 * u + 2] = o[1];
      v0[4 * u + 3] = o[3];
      v1[4 * u + 0] = o[4];
      v1[4 * u + 1] = o[6];
      v1[4 * u + 2] = o[5];
      v1[4 * u + 3] = o[7];
    }
    tmem_st16x256_x4(taddr + (uint32_t)(nm * 64), v0);  // A block nm: 64 columns (128 k)
    tmem_st16x256_x4(taddr + (16u << 16) + (uint32_t)(nm * 64), v1);
  }
}

// ---------------------------------------------------------------- the kernel
// Persistent: CTA c handles items c, c + grid, ...  Three rings decouple the
// roles: packed weights (deep, HBM latency), dequantized A, activation images.
// Every role walks the same stage sequence: per item, k / 128 main stages then
// the LoRC stages of each 64-rank chunk per matrix.
#ifndef PF_SPIN_WAITS
#define PF_SPIN_WAITS 0  // experiments: all ring waits spin on test_wait instead of try_wait
#endif
__device__ __forceinline__ void ring_wait(uint64_t* bar, uint32_t parity) {
  if (PF_SPIN_WAITS)
    pf_wait(bar, parity);
  else
    mbar_wait(bar, parity);
}
template <int NMAT, int NG>
__global__ void __launch_bounds__(PfRoles<NMAT, NG>::kThreads, 1) pf_gemm_kernel(const __grid_constant__ PfArgs a_in) {
  PfArgs a = a_in;
  if (a.dev_counts != nullptr) {  // planned on the device: sizes from the plan
    a.n_problems = a.dev_counts[0];
    a.n_items = a.dev_counts[1];
    a.ntok_max = a.dev_counts[2];
  }

  constexpr int kPfDeqGroups = PfRoles<NMAT, NG>::kGroups;
  static_assert(kPfDeqGroups <= 4, "dequant groups must not outnumber A slots (>= 4)");
  using CF = PfCfg<NMAT, NG>;
  constexpr int PS = CF::kPS;
  const int bslot = 2 * a.ntok_max * 128;
  const int BS = min(CF::kBSMax, CF::kBRegion / bslot);
  // accumulators: per matrix a 32-column-aligned block of ntok_max columns;
  // two buffers when both fit the 256 accumulator columns
  const int mstride = (a.ntok_max + 31) & ~31;
  // one accumulator per (n-tile, matrix); a single-accumulator kernel with
  // small token tiles splits each stage's k over two accumulators (one per
  // MMA issuer, summed by the epilogue)
  const bool ksplit = false;  // (a two-issuer k split of one-matrix items measured slower)
  const int acc_cols = (ksplit ? 2 : NG * NMAT) * mstride;
  // TMEM columns: accumulators (double-buffered when that leaves >= PF_MIN_AS
  // A slots), then the A slots (128-k stages: 3 slots for two matrices at 64
  // tokens with one accumulator buffer; double buffering with 2 measured equal).
  const int nacc = (acc_cols <= 128 && (512 - 2 * acc_cols) / CF::kStageCols >= PF_MIN_AS) ? 2 : 1;
  const int a_col0 = nacc * acc_cols;
  const int AS = min(CF::kASMax, (512 - a_col0) / CF::kStageCols);
  // parity waits on the A ring are unambiguous only with at least as many slots as
  // dequant groups (a smaller ring would deadlock): fail loudly instead
  if (AS < kPfDeqGroups) __trap();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned base (SW128 atoms); pointer arithmetic keeps the shared address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::kOffBar);
  uint64_t* p_full = bars;
  uint64_t* p_empty = p_full + PS;
  uint64_t* a_full = p_empty + PS;
  uint64_t* a_empty = a_full + CF::kASMax;
  uint64_t* b_full = a_empty + CF::kASMax;
  uint64_t* b_empty = b_full + CF::kBSMax;
  uint64_t* acc_full = b_empty + CF::kBSMax;  // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + CF::kOffTmem);
  uint32_t* stages_ready = tmem_slot + 1;  // kPfWaitWarp -> MMA issuers: stages whose A and B are in place
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < PS; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&p_empty[s], kPfGroupWarps);  // the group of the slot's stage
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(&a_full[s], kPfGroupWarps);
      mbar_init(&a_empty[s], 2);  // one commit (or arrive) per MMA issuer
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 2);
      mbar_init(&acc_empty[i], kPfEpiWarps);
    }
    *stages_ready = 0;
    fence_barrier_init();
  }
  if (warp == kPfMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  auto pf_dbg = [&](int i) {
    if (a.dbg != nullptr) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.dbg[blockIdx.x * 8 + i] = t;
    }
  };
  if (threadIdx.x == 0) pf_dbg(0);
  // CTA 0, first kPfTraceStages stages of its whole sequence: [stage][8 events]
  //   0 packed issued  1 group: A slot free  2 group: packed landed  3 group: A ready
  //   4 MMA: A seen    5 MMA: B seen         6 MMA: committed        7 B issued
  auto pf_trace = [&](int stage, int ev) {
    if (a.dbg != nullptr && blockIdx.x == 0 && stage < kPfTraceStages) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.dbg[148 * 8 + stage * 8 + ev] = t;
    }
  };

  // stages: main stages of 128 k (P.k % 128 == 0), then the LoRC stages per 64-rank
  // chunk per matrix.  Merged (token tiles >= PF_LMERGE_MIN): one stage, V^T hi | lo
  // in the A slot, t hi | lo in the B slot, three MMA passes (hi.hi + hi.lo + lo.hi).
  // Else three stages of one pass each (V_hi.t_hi, V_hi.t_lo, V_lo.t_hi): for small
  // tiles the stage is latency-bound and splitting it spreads it over both groups.
  auto lmerged = [&](const PfProblem& P) { return PF_LMERGE_MIN <= kPfN && P.ntok >= PF_LMERGE_MIN; };
  auto item_stages = [&](const PfProblem& P) {
    return P.k / (2 * kPfK) + (lmerged(P) ? 1 : 3) * (P.rchunks[0] + (NMAT == 2 ? P.rchunks[1] : 0));
  };
  // LoRC stage l (0-based after the main stages) -> matrix, chunk, V part, t part
  // (part -1: both, merged stage)
  auto lorc_stage = [&](const PfProblem& P, int l, int& mat, int& ch, int& vpart, int& tpart) {
    const int per = lmerged(P) ? 1 : 3;
    mat = 0;
    if (l >= per * P.rchunks[0]) {
      l -= per * P.rchunks[0];
      mat = 1;
    }
    ch = l / per;
    const int part = l % per;  // 0: V_hi.t_hi, 1: V_hi.t_lo, 2: V_lo.t_hi
    vpart = per == 1 ? -1 : (part == 2 ? 1 : 0);
    tpart = per == 1 ? -1 : (part == 1 ? 1 : 0);
  };

#if PF_PROF  // per-role cycle split, CTA 0 -> dbg trace row kPfTraceStages - 1 - role
  long long pf_prof[4] = {0, 0, 0, 0};
  long long pf_t0 = clock64();
#define PF_LAP(i)                    \
  do {                               \
    const long long t_ = clock64();  \
    pf_prof[i] += t_ - pf_t0;        \
    pf_t0 = t_;                      \
  } while (0)
#define PF_PROF_OUT(role)                                                                         \
  if (a.dbg != nullptr && blockIdx.x == 0)                                                        \
    for (int i = 0; i < 4; ++i) a.dbg[148 * 8 + (kPfTraceStages - 1 - (role)) * 8 + i] = pf_prof[i]
#else
#define PF_LAP(i)
#define PF_PROF_OUT(role)
#endif
  if (warp == kPfProdWarp) {
    // ======================= packed-weight producer =======================
    // A stage's NG x NMAT x 2 copies are issued by as many lanes in parallel: one
    // thread serialises its bulk copies at ~300 cycles each (tools/micro/bulk_issue.cu).
    constexpr int kCopies = NG * NMAT * 2;  // one 4-k-tile run of one slab each
    if (lane < kCopies) {
      const int ng = lane / (NMAT * 2), mat = (lane / 2) % NMAT, sl = lane & 1;
      int ps = 0, gs0 = 0;
      uint32_t pph = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        int p, nt, tt;
        pf_item<NG>(a, item, p, nt, tt);
        const PfProblem P = a.problems[p];  // by value: fields live in registers
        const int ks2 = P.k / (2 * kPfK), kts = P.k / kTileK;
        // the item's V^T images (its LoRC stages come last) -> L2 now: one contiguous
        // run of rchunks x (hi, lo) images per (n-tile, matrix)
        if (PF_VPREFETCH && lane < NG * NMAT && P.rchunks[lane % NMAT] > 0) {
          const int pm = lane % NMAT, png = lane / NMAT;
          const uint32_t run = (uint32_t)P.rchunks[pm] * 2u * kPfImg;
          prefetch_l2(P.vimg[pm] + (int64_t)(NG * nt + png) * run, run);
        }
        for (int sp = 0; sp < ks2; ++sp) {
          ring_wait(&p_empty[ps], pph ^ 1);
          PF_LAP(0);
          uint8_t* sP = smem + CF::kOffP + ps * CF::kStageP;
          if (lane == 0) mbar_arrive_expect_tx(&p_full[ps], (uint32_t)CF::kStageP);
          __syncwarp((1u << kCopies) - 1u);
          const int kp = (sp + nt * 13) % ks2;  // rotated k order per n-tile (spreads L2 hot spots)
          const uint8_t* src = P.w[mat] + ((int64_t)(2 * (NG * nt + ng) + sl) * kts + 4 * kp) * kTileBytes;
          bulk_g2s(sP + ((ng * NMAT + mat) * 2 + sl) * 4 * kTileBytes, src, 4 * kTileBytes, &p_full[ps]);
          if (lane == 0) pf_trace(gs0 + sp, 0);
          PF_LAP(1);
          if (++ps == PS) {
            ps = 0;
            pph ^= 1;
          }
        }
        gs0 += item_stages(P);
      }
      if (lane == 0) {
        PF_PROF_OUT(3);
        pf_dbg(1);
      }
    }
  } else if (warp == kPfBWarp) {
    // ======================= activation / t image producer =======================
    // one copy per main-stage pair (the two 64-k images of a token tile are
    // adjacent), one per LoRC stage
    if (lane == 0) {
      int bs = 0, gs = 0;
      uint32_t bph = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        int p, nt, tt;
        pf_item<NG>(a, item, p, nt, tt);
        const PfProblem P = a.problems[p];  // by value: fields live in registers
        const int ks = P.k / (2 * kPfK), total = item_stages(P);
        const uint32_t ib = (uint32_t)P.ntok * 128u;  // one token-tile image (64 k)
        for (int st = 0; st < total; ++st, ++gs) {
          ring_wait(&b_empty[bs], bph ^ 1);
          PF_LAP(0);
          uint8_t* sB = smem + CF::kOffB + bs * bslot;
          const uint8_t* src;
          uint32_t bytes = ib;
          if (st < ks) {  // the two adjacent 64-k images of the stage
            const int kp = (st + nt * 13) % ks;  // same rotation as the weights
            src = P.act + ((int64_t)tt * 2 * ks + 2 * kp) * ib;
            bytes = 2 * ib;
          } else {  // t hi / lo image of the chunk (merged: both, adjacent)
            int mat, ch, vpart, tpart;
            lorc_stage(P, st - ks, mat, ch, vpart, tpart);
            src = P.timg[mat] + (((int64_t)tt * P.rchunks[mat] + ch) * 2 + (tpart > 0 ? 1 : 0)) * ib;
            bytes = tpart < 0 ? 2 * ib : ib;
          }
          mbar_arrive_expect_tx(&b_full[bs], bytes);
          bulk_g2s(sB, src, bytes, &b_full[bs]);
          pf_trace(gs, 7);
          PF_LAP(1);
          if (++bs == BS) {
            bs = 0;
            bph ^= 1;
          }
        }
      }
      PF_PROF_OUT(2);
      pf_dbg(2);
    }
  } else if (warp >= kPfDeqWarp0 && warp < kPfDeqWarp0 + PfRoles<NMAT, NG>::kDeqWarps) {
    // ======================= dequant warps =======================
    // group grp handles the stages st = grp (mod kPfDeqGroups); within a stage,
    // warp w writes TMEM lane quarter Q = w % 4 (the only lanes its tcgen05.st
    // can reach): A rows 32 Q .. 32 Q + 31 = slab Q / 2, n subtiles i of half
    // Q % 2 -- half of every unit of that slab (half_unit_dequant).  Main stage:
    // packed tiles -> bit-exact binary16 W^T -> tcgen05.st.16x256b, k pair
    // (q, q + 4) of each 16-k block into columns (2q, 2q + 1) (the activation
    // images carry the same permutation, pf_image_kernel).  LoRC stage: the
    // V^T image rows of the quarter (L2-resident) -> tcgen05.st.32x32b.
    const int dw = warp - kPfDeqWarp0;
    const int grp = dw / kPfGroupWarps, gw = dw % kPfGroupWarps;
    const int Q = warp & 3, sl = Q >> 1, ih = Q & 1;
    const int q = lane & 3;
    const uint32_t lane_q = (uint32_t)(32 * Q) << 16;
    int ps = 0, as = 0, gs = 0;
    uint32_t pph = 0, aph = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      int p, nt, tt;
      pf_item<NG>(a, item, p, nt, tt);
      const PfProblem P = a.problems[p];  // by value: fields live in registers
      const int ks = P.k / (2 * kPfK), total = item_stages(P);
      const DqConsts dq = make_dq_consts(P.mode);
      for (int st = 0; st < total; ++st, ++gs) {
        const bool mine = (gs % kPfDeqGroups) == grp;
        if (mine) {
          const uint32_t a_col = tmem + (uint32_t)(a_col0 + as * CF::kStageCols);
          PF_LAP(3);  // (not this group's stages)
          ring_wait(&a_empty[as], aph ^ 1);  // the MMAs that read this slot are done
          PF_LAP(0);
          tc_fence_after();
          if (gw == 0 && lane == 0) pf_trace(gs, 1);
          if (st < ks) {
            ring_wait(&p_full[ps], pph);
            PF_LAP(1);
            if (gw == 0 && lane == 0) pf_trace(gs, 2);
            // the slot's [nm][slab][4 k-tiles] runs: k-tiles 0, 1 -> A columns nm * 64 + [0, 32),
            // k-tiles 2, 3 -> nm * 64 + [32, 64)
            const uint8_t* sP = smem + CF::kOffP + ps * CF::kStageP + sl * 4 * kTileBytes;
            if (!(a.flags & 1)) {  // branch-free stage bodies per half (the units interleave)
#if PF_DQ_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
              for (int h = 0; h < 2; ++h) {
                if (ih == 0)
                  pf_dequant_stage<0, NG * NMAT>(sP + h * 2 * kTileBytes, lane, dq, a_col + lane_q + 32 * h);
                else
                  pf_dequant_stage<1, NG * NMAT>(sP + h * 2 * kTileBytes, lane, dq, a_col + lane_q + 32 * h);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_empty[ps]);
          } else {
            int mat, ch, vp, tp;
            lorc_stage(P, st - ks, mat, ch, vp, tp);
            const int row = 32 * Q + lane, nv = vp < 0 ? 2 : 1;
#pragma unroll 1
            for (int ngv = 0; ngv < nv * NG; ++ngv) {  // (n-tile, V part): merged V hi -> columns [0, 32), lo -> [32, 64)
              const int ng = ngv / nv, vpart = vp < 0 ? (ngv & 1) : vp;
              const uint8_t* img =
                  P.vimg[mat] + (((int64_t)(NG * nt + ng) * P.rchunks[mat] + ch) * 2 + vpart) * kPfImg + row * 128;
              uint32_t v[32];
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const uint4 x = __ldg(reinterpret_cast<const uint4*>(img + ((c ^ (row & 7)) << 4)));
                v[4 * c] = x.x;
                v[4 * c + 1] = x.y;
                v[4 * c + 2] = x.z;
                v[4 * c + 3] = x.w;
              }
              tmem_st32x32_x32(a_col + lane_q + (uint32_t)((ng * NMAT + mat) * 64 + (vp < 0 ? 32 * vpart : 0)), v);
            }
          }
          PF_LAP(2);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_full[as]);
          if (gw == 0 && lane == 0) pf_trace(gs, 3);
        }
        if (st < ks && ++ps == PS) {
          ps = 0;
          pph ^= 1;
        }
        if (++as == AS) {
          as = 0;
          aph ^= 1;
        }
      }
    }
    if (dw == 0 && lane == 0) {
      PF_PROF_OUT(4);
      pf_dbg(3);
    }
  } else if (warp == kPfWaitWarp) {
    // ======================= ring waiter =======================
    if (lane == 0) {
      int as = 0, bs = 0, gs = 0;
      uint32_t aph = 0, bph = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        int p, nt, tt;
        pf_item<NG>(a, item, p, nt, tt);
        const int total = item_stages(a.problems[p]);
        for (int st = 0; st < total; ++st, ++gs) {
          ring_wait(&a_full[as], aph);
          PF_LAP(0);
          pf_trace(gs, 4);
          ring_wait(&b_full[bs], bph);
          PF_LAP(1);
          pf_trace(gs, 5);
          st_release_cta_shared(stages_ready, (uint32_t)(gs + 1));
          PF_LAP(2);
          if (++as == AS) {
            as = 0;
            aph ^= 1;
          }
          if (++bs == BS) {
            bs = 0;
            bph ^= 1;
          }
        }
      }
      PF_PROF_OUT(1);
    }
  } else if (warp == kPfMmaWarp || warp == kPfMmaWarp2) {
    // ======================= MMA issuers =======================
    // Two threads issue (a single thread issues at most one tcgen05.mma per
    // ~55 cycles, tools/micro/mma_rate.cu, while a 128 x 64 x 16 MMA executes
    // in 32): issuer i owns accumulator i -- matrix i (w1 / w3), n-tile i, or
    // for one-accumulator kernels with ntok <= 64 the k16 steps i, i + 2 of
    // every stage.  Both release every A / B slot (commit, or a plain arrive
    // when the stage has no MMA of theirs) and every accumulator.
    const int issuer = warp == kPfMmaWarp ? 0 : 1;
    {  // the whole warp (converged), one elected lane issues
      const uint64_t dB0 = pf_desc_sw128(smem_u32(smem + CF::kOffB));
      const bool mma_on = !(a.flags & 2);
      int as = 0, bs = 0;
      int acc = 0, gs = 0;
      uint32_t acc_phase = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        int p, nt, tt;
        pf_item<NG>(a, item, p, nt, tt);
        const PfProblem P = a.problems[p];  // by value: fields live in registers
        const int ks = P.k / (2 * kPfK), total = item_stages(P);
        const uint32_t idesc = pf_idesc(P.ntok);
        const uint32_t ib16 = ((uint32_t)P.ntok * 128u) >> 4;  // one image, in descriptor units
        ring_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + (uint32_t)(acc * acc_cols);  // accumulator buffer
        const bool idle = (PF_ISSUERS == 1 || (NG * NMAT == 1 && !ksplit)) && issuer == 1;
        for (int st = 0; st < total; ++st, ++gs) {
          // an mbarrier wait costs a thread that issues MMAs ~200 cycles even when
          // the phase completed long ago (tools/micro/mma_rate.cu); the wait warp
          // does the ring waits and publishes a stage counter instead
          while (ld_acquire_cta_shared(stages_ready) <= (uint32_t)gs) {
          }
          PF_LAP(0);
          tc_fence_after();
          // operand addresses: TMEM A slot, B descriptor of the slot (the 16-B
          // address field advances by 2 per 16-k step); everything unrolled
          const uint32_t aA = tmem + (uint32_t)(a_col0 + as * CF::kStageCols);
          // B: the slot's two 64-k images (main stage) or its t image
          const uint64_t dB = dB0 + (uint64_t)((uint32_t)(bs * bslot) >> 4);
          bool issued = false;
          if (!idle && mma_on) {
            uint32_t acc0 = 1u;
            int lmat = -1, ltp = -1;  // LoRC stage: its matrix, t part (-1 merged)
            if (st < ks) {
              acc0 = st > 0 ? 1u : 0u;
            } else {
              int ch, vp;
              lorc_stage(P, st - ks, lmat, ch, vp, ltp);
            }
#if PF_ISSUE_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
            for (int nm = 0; nm < NG * NMAT; ++nm) {  // A block (ng * NMAT + mat) = accumulator nm
              if (PF_ISSUERS == 2 && nm % 2 != issuer) continue;
              if (lmat >= 0 && nm % NMAT != lmat) continue;  // LoRC: that matrix's blocks only
              const uint32_t dN = d0 + (uint32_t)(nm * mstride), aN = aA + (uint32_t)(nm * 64);
              if (st < ks) {  // 8 k16 steps: image 0 then image 1 of the slot
#pragma unroll
                for (int k16 = 0; k16 < 8; ++k16)
                  pf_mma_ts_w(dN, aN + (uint32_t)(k16 * 8), dB + (k16 < 4 ? 2 * k16 : ib16 + 2 * (k16 - 4)), idesc,
                              k16 > 0 ? 1u : acc0);
              } else if (ltp >= 0) {  // LoRC part, 64 ranks: 4 k16 steps (t part ltp)
#pragma unroll 1
                for (int k16 = 0; k16 < 4; ++k16) pf_mma_ts_w(dN, aN + (uint32_t)(k16 * 8), dB + 2 * k16, idesc, 1u);
              } else {  // merged LoRC, 64 ranks: V_hi.t_hi + V_hi.t_lo + V_lo.t_hi
#pragma unroll 1
                for (int k16 = 0; k16 < 4; ++k16) {
                  pf_mma_ts_w(dN, aN + (uint32_t)(k16 * 8), dB + 2 * k16, idesc, 1u);
                  pf_mma_ts_w(dN, aN + (uint32_t)(k16 * 8), dB + ib16 + 2 * k16, idesc, 1u);
                  pf_mma_ts_w(dN, aN + (uint32_t)(32 + k16 * 8), dB + 2 * k16, idesc, 1u);
                }
              }
              issued = true;
            }
          }
          PF_LAP(1);
          if (issued) {
            pf_commit_w(&a_empty[as]);
            pf_commit_w(&b_empty[bs]);
          } else {
            mbar_arrive_w(&a_empty[as]);
            mbar_arrive_w(&b_empty[bs]);
          }
          if (++bs == BS) bs = 0;
          PF_LAP(2);
          if (issuer == 0 && lane == 0) pf_trace(gs, 6);
          if (++as == AS) as = 0;
        }
        if (idle || !mma_on)
          mbar_arrive_w(&acc_full[acc]);
        else
          pf_commit_w(&acc_full[acc]);
        if (++acc == nacc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (issuer == 0 && lane == 0) {
        PF_PROF_OUT(0);
        pf_dbg(4);
      }
    }
  } else {
    // ======================= epilogue warps =======================
    // quarter ew: TMEM lanes 32 ew .. 32 ew + 31 = A rows (output columns); with two
    // warps per quarter they take alternate 16-token passes
    const int ew = warp & 3, eh = warp < 4 ? 0 : 1;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      int p, nt, tt;
      pf_item<NG>(a, item, p, nt, tt);
      const PfProblem P = a.problems[p];  // by value: fields live in registers
      PF_LAP(2);
      ring_wait(&acc_full[acc], acc_phase);
      PF_LAP(0);
      tc_fence_after();
      if (threadIdx.x == 0) pf_dbg(6);
      // TMEM -> registers (thread = output column, 32 tokens per load) -> SwiGLU /
      // identity -> smem transpose -> 16-byte row stores (8 token rows per instruction)
      const int rows = P.rows, kind = P.kind, odt = P.out_dtype;
      const int64_t ldo = P.ldo;
      const int32_t* rmap = P.row_map;
      float* stg = reinterpret_cast<float*>(smem + CF::kOffStage) + (ew + 4 * eh) * 16 * 33;
      const int ntok = P.ntok;
#pragma unroll 1
      for (int ng = 0; ng < NG; ++ng) {
      const uint32_t tbase = tmem + ((uint32_t)(32 * ew) << 16) + (uint32_t)(acc * acc_cols + ng * NMAT * mstride);
      const int col0 = (NG * nt + ng) * kPfM + 32 * ew + 8 * (lane & 3);  // this lane's 8 output columns
#pragma unroll 1
      for (int c0 = 16 * eh; c0 < ntok; c0 += 16 * PF_EPI_HALVES) {  // 16 tokens per pass
        uint32_t v0[16], v1[16];
        tmem_ld16(tbase + (uint32_t)c0, v0);
        if (NMAT == 2 || ksplit) tmem_ld16(tbase + (uint32_t)(mstride + c0), v1);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float x = __uint_as_float(v0[c]);
          if (NMAT == 1 && ksplit) x += __uint_as_float(v1[c]);  // the two k halves
          if (kind == 1) x = pf_silu(x) * (NMAT == 2 ? __uint_as_float(v1[c]) : 0.0f);
          stg[c * 33 + lane] = x;
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 2; ++it) {
          const int tr = 8 * it + (lane >> 2);  // token row within the chunk
          const int row = tt * ntok + c0 + tr;
          if (row < rows && c0 + tr < ntok) {
            const int64_t orow = rmap ? rmap[row] : row;
            const float* src = stg + tr * 33 + 8 * (lane & 3);
            float f[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) f[u] = src[u];
            if (kind == 0 && odt == 0) {
              float4* dst = reinterpret_cast<float4*>(static_cast<float*>(P.out) + orow * ldo + col0);
              dst[0] = make_float4(f[0], f[1], f[2], f[3]);
              dst[1] = make_float4(f[4], f[5], f[6], f[7]);
            } else {
              uint4 h;
              h.x = h2_as_u32(__floats2half2_rn(f[0], f[1]));
              h.y = h2_as_u32(__floats2half2_rn(f[2], f[3]));
              h.z = h2_as_u32(__floats2half2_rn(f[4], f[5]));
              h.w = h2_as_u32(__floats2half2_rn(f[6], f[7]));
              *reinterpret_cast<uint4*>(static_cast<__half*>(P.out) + orow * ldo + col0) = h;
            }
          }
        }
        __syncwarp();
      }
      }  // ng
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      PF_LAP(1);
      if (++acc == nacc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (warp == 0 && lane == 0) PF_PROF_OUT(5);
  }
  if (threadIdx.x == 0) pf_dbg(5);
  __syncthreads();
  if (warp == kPfMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(CF::kTmemCols));
  }
  pdl_launch_dependents();
}

// Activation images: rows (binary16 or f32 source, optional row gather) ->
// [tok_tiles][k/64][ntok rows x 128 B, SW128 K-major], zero rows past `rows`.
// Within every 16-k block the k pairs are stored in the order 0 4 1 5 2 6 3 7
// -- the column order in which pf_gemm_kernel's dequant warps write W^T into
// tensor memory (thread q of a quad owns pairs q and q + 4 of the mma
// fragment and stores them to adjacent columns 2q, 2q + 1).
// One 16-k block (8 pairs w[0..7]) of row src_row at column col.
__device__ __forceinline__ void pf_load_block16(const void* x, int32_t x_dtype, int64_t src_row, int64_t ldx,
                                                int64_t col, uint32_t (&w)[8]) {
  if (x_dtype == 0) {
    const float4* s = reinterpret_cast<const float4*>(static_cast<const float*>(x) + src_row * ldx + col);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 f = s[u];
      w[2 * u] = h2_as_u32(__floats2half2_rn(f.x, f.y));
      w[2 * u + 1] = h2_as_u32(__floats2half2_rn(f.z, f.w));
    }
  } else {
    const uint4* s = reinterpret_cast<const uint4*>(static_cast<const __half*>(x) + src_row * ldx + col);
    const uint4 p0 = s[0], p1 = s[1];
    w[0] = p0.x; w[1] = p0.y; w[2] = p0.z; w[3] = p0.w;
    w[4] = p1.x; w[5] = p1.y; w[6] = p1.z; w[7] = p1.w;
  }
}
// Stores block b (0..3) of image row r in the permuted order.
__device__ __forceinline__ void pf_store_block16(uint8_t* dst, int r, int b, const uint32_t (&w)[8]) {
  *reinterpret_cast<uint4*>(dst + r * 128 + (((2 * b) ^ (r & 7)) << 4)) = make_uint4(w[0], w[4], w[1], w[5]);
  *reinterpret_cast<uint4*>(dst + r * 128 + (((2 * b + 1) ^ (r & 7)) << 4)) = make_uint4(w[2], w[6], w[3], w[7]);
}
__global__ void pf_image_kernel(const void* __restrict__ x, int32_t x_dtype, int64_t ldx,
                                const int32_t* __restrict__ row_ids, int32_t rows, int32_t k, int32_t ntok,
                                uint8_t* __restrict__ img) {
  const int ks = k / kPfK;
  const int tile = blockIdx.x / ks, st = blockIdx.x % ks;
  uint8_t* dst = img + (int64_t)blockIdx.x * ntok * 128;
  for (int c = threadIdx.x; c < ntok * 4; c += blockDim.x) {  // 16-k blocks
    const int r = c >> 2, b = c & 3;
    const int row = tile * ntok + r;
    uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if (row < rows) pf_load_block16(x, x_dtype, row_ids ? row_ids[row] : row, ldx, (int64_t)st * kPfK + b * 16, w);
    pf_store_block16(dst, r, b, w);
  }
  pdl_launch_dependents();
}

}  // namespace milo_dev

namespace milo_dev {

// ---------------------------------------------------------------------------
// LoRC for the prefill path: t = half(X) U on the CUDA cores (fp32, like the
// reference's Eigen product, gemm.cpp:185-188), split over k and reduced in a
// fixed order, then written as binary16 hi / lo operand images for the GEMM's
// extra K stages (t V on the tensor cores).
// ---------------------------------------------------------------------------
struct TProb {
  const void* x;            // activation rows (f32 or f16)
  int32_t x_dtype;
  int64_t ldx;
  const int32_t* row_ids;   // x row of problem row r (null: r)
  int32_t rows, k, rank, gpr, rchunks, ks;  // ks = k splits
  const uint8_t* ucodes;    // k x rank symm-int3 codes (or null -> ureal)
  const float* uscales;     // k x gpr
  const float* ureal;       // k x rank
  float* part;              // [ks][rows][rchunks * 64] fp32 partials
  uint8_t* timg;            // [tok_tiles][rchunks][hi, lo][ntok x 128 B]
  int32_t ntok;
  int32_t unit0;            // first work unit of this problem (prefix)
};

#ifndef PF_T_CTAS
#define PF_T_CTAS 2  // t-kernel k splits target ~2 units per SM (4 CTAs per SM resident)
#endif
constexpr int kTRows = 32;  // rows per t-kernel CTA
constexpr int kTCtasPerSm = PF_T_CTAS;

// One k block of pf_t_kernel's operands into registers: x (binary16-rounded)
// at column lc of rows lr + 4 i, U = step (c - 4) (lowrank.cpp:122-134) or the
// real factor at k-rows lr + 4 i.  Every load is issued before any is consumed.
__device__ __forceinline__ void t_load_block(const TProb& P, int kb, int lc, int lr, int ch, int urc, bool uok,
                                             const int64_t (&xrow)[8], float (&xv)[8], float (&uv)[16]) {
  if (P.x_dtype == 0) {
    const float* xp = static_cast<const float*>(P.x) + kb + lc;
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = xrow[i] >= 0 ? __half2float(__float2half_rn(xp[xrow[i]])) : 0.0f;
  } else {
    const __half* xp = static_cast<const __half*>(P.x) + kb + lc;
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = xrow[i] >= 0 ? __half2float(xp[xrow[i]]) : 0.0f;
  }
  if (P.ucodes) {
    const uint8_t* cp = P.ucodes + (int64_t)(kb + lr) * P.rank + urc;
    const float* sp = P.uscales + (int64_t)(kb + lr) * P.gpr + ch;
    uint32_t c[16];
    float st[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      c[i] = uok ? cp[(int64_t)4 * i * P.rank] : 4u;
      st[i] = uok ? sp[(int64_t)4 * i * P.gpr] : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) uv[i] = (st[i] * (2.0f / 7.0f)) * ((float)c[i] - 4.0f);
  } else {
    const float* rp = P.ureal + (int64_t)(kb + lr) * P.rank + urc;
#pragma unroll
    for (int i = 0; i < 16; ++i) uv[i] = uok ? rp[(int64_t)4 * i * P.rank] : 0.0f;
  }
}

// One unit (problem, token tile, rank chunk, k split) of pf_t_kernel.
__device__ __forceinline__ void pf_t_unit(const TProb* __restrict__ probs, int n_probs, int unit,
                                          float (&sx)[kTRows][68], float (&su)[64][65]) {
  int lo = 0, hi = n_probs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (probs[mid].unit0 <= unit) lo = mid; else hi = mid - 1;
  }
  const TProb& P = probs[lo];
  int u = unit - P.unit0;
  const int tiles = (P.rows + kTRows - 1) / kTRows;
  const int ksi = u % P.ks;
  u /= P.ks;
  const int ch = u % P.rchunks, tile = u / P.rchunks;
  if (tile >= tiles) return;
  const int kper = ((P.k / 64 + P.ks - 1) / P.ks) * 64;
  const int k0 = ksi * kper, k1 = min(P.k, k0 + kper);
  const int tid = threadIdx.x, j = tid & 63, rg = tid >> 6;  // rank column, row group (8 rows)
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
  const int rcol = ch * 64 + j;
  // Loader role: column lc of x rows lr + 4 i and of U k-rows lr + 4 i (the x
  // row bases resolved once).  (Prefetching block kb + 64 into registers during
  // the product measured slower: 112 registers, one CTA per SM either way.)
  const int lc = tid & 63, lr = tid >> 6;
  int64_t xrow[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = tile * kTRows + lr + 4 * i;
    xrow[i] = row < P.rows ? (P.row_ids ? (int64_t)P.row_ids[row] : (int64_t)row) * P.ldx : int64_t(-1);
  }
  const int urc = ch * 64 + lc;
  const bool uok = urc < P.rank;
  float xv[8], uv[16];
  if (k0 < k1) t_load_block(P, k0, lc, lr, ch, urc, uok, xrow, xv, uv);
  for (int kb = k0; kb < k1; kb += 64) {
#pragma unroll
    for (int i = 0; i < 8; ++i) sx[lr + 4 * i][lc] = xv[i];
#pragma unroll
    for (int i = 0; i < 16; ++i) su[lr + 4 * i][lc] = uv[i];
    __syncthreads();
    // Shared-load bound: x read as float4 (4 k per read; per-k summation order
    // unchanged), and warps whose 32 rank columns all lie past the rank skip the
    // product (every rank <= 32 leaves half the CTA idle otherwise).
    if (ch * 64 + (j & ~31) < P.rank) {
#pragma unroll 2
      for (int kk = 0; kk < 64; kk += 4) {
        const float u0 = su[kk][j], u1 = su[kk + 1][j], u2 = su[kk + 2][j], u3 = su[kk + 3][j];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 xq = *reinterpret_cast<const float4*>(&sx[rg * 8 + i][kk]);
          acc[i] += xq.x * u0;
          acc[i] += xq.y * u1;
          acc[i] += xq.z * u2;
          acc[i] += xq.w * u3;
        }
      }
    }
    __syncthreads();
    if (kb + 64 < k1) t_load_block(P, kb + 64, lc, lr, ch, urc, uok, xrow, xv, uv);
  }
  const int r64 = P.rchunks * 64;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = tile * kTRows + rg * 8 + i;
    if (row < P.rows) P.part[((int64_t)ksi * P.rows + row) * r64 + rcol] = acc[i];
  }
}

// The same unit for symm-INT3 factors on the tensor cores (mma.sync
// m16n8k16, fp32 accumulation): U[k][j] = s'[k] (c[k][j] - 4) with
// s' = scale x 2/7 per (k, 64-rank group) (lowrank.cpp:122-134), so
//   t = half(x) U = (half(x) (.) s') C,   C = c - 4 exact in binary16,
// and the fp32 row-scaled activations p = half(x) s' enter as binary16 hi + lo
// halves (p - hi(p) is exact in fp32; hi + lo carries 22 of its 24 bits).  The
// products with C are exact and accumulate in fp32 -- the reference's fp32
// product up to summation order and the 2^-22 split residual.
struct TTcSmem {
  __half xh[kTRows][72];  // p hi, rows of the tile x 64 k (+8 pad: conflict-free fragment loads)
  __half xl[kTRows][72];  // p lo
  __half ct[64][72];      // C^T: 64 ranks x 64 k
};
__device__ __forceinline__ void t_tc_load(const TProb& P, int kb, int ch, int tid, const int64_t xrow, float (&xv)[8],
                                          float (&sv)[8], uint4& cv) {
  const int k8 = (tid & 7) * 8;  // x: row tid / 8, k k8 .. k8 + 7
  if (xrow >= 0) {
    if (P.x_dtype == 0) {
      const float4* xp = reinterpret_cast<const float4*>(static_cast<const float*>(P.x) + xrow + kb + k8);
      const float4 a = xp[0], b = xp[1];
      const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) xv[i] = __half2float(__float2half_rn(f[i]));
    } else {
      const uint4 h = *reinterpret_cast<const uint4*>(static_cast<const __half*>(P.x) + xrow + kb + k8);
      const uint32_t w[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(u32_as_h2(w[i]));
        xv[2 * i] = f.x;
        xv[2 * i + 1] = f.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = 0.0f;
  }
  if (P.gpr == 1) {
    const float4* sp = reinterpret_cast<const float4*>(P.uscales + kb + k8);
    const float4 a = __ldg(sp), b = __ldg(sp + 1);
    sv[0] = a.x; sv[1] = a.y; sv[2] = a.z; sv[3] = a.w;
    sv[4] = b.x; sv[5] = b.y; sv[6] = b.z; sv[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) sv[i] = P.uscales[(int64_t)(kb + k8 + i) * P.gpr + ch];
  }
  if (P.rchunks == 1) {
    // the block's codes are one contiguous run of 64 x rank bytes (16-B aligned:
    // 64 rank is): thread tid loads bytes 16 tid .. 16 tid + 15 of it
    const int nb = 64 * P.rank;
    cv = 16 * tid < nb ? __ldg(reinterpret_cast<const uint4*>(P.ucodes + (int64_t)kb * P.rank + 16 * tid))
                       : make_uint4(0u, 0u, 0u, 0u);
  } else if (P.rank % 16 == 0) {
    // codes: k row tid / 4, ranks ch * 64 + 16 (tid % 4) .. + 15: one aligned 16-B load
    const int kk = tid >> 2, j0 = ch * 64 + (tid & 3) * 16;
    cv = j0 < P.rank ? __ldg(reinterpret_cast<const uint4*>(P.ucodes + (int64_t)(kb + kk) * P.rank + j0))
                     : make_uint4(0x04040404u, 0x04040404u, 0x04040404u, 0x04040404u);
  } else {
    // codes: k row tid / 4, ranks ch * 64 + 16 (tid % 4) .. + 15 (past the rank: code 4 -> 0)
    const int kk = tid >> 2, j0 = ch * 64 + (tid & 3) * 16;
    const uint8_t* cp = P.ucodes + (int64_t)(kb + kk) * P.rank + j0;
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = j0 + 4 * i + b;
        const uint32_t c = j < P.rank ? cp[4 * i + b] : 4u;
        v |= c << (8 * b);
      }
      w[i] = v;
    }
    cv = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
__device__ __forceinline__ void pf_t_tc_unit(const TProb& P, int u, TTcSmem& sm) {
  const int tiles = (P.rows + kTRows - 1) / kTRows;
  const int ksi = u % P.ks;
  u /= P.ks;
  const int ch = u % P.rchunks, tile = u / P.rchunks;
  if (tile >= tiles) return;
  const int kper = ((P.k / 64 + P.ks - 1) / P.ks) * 64;
  const int k0 = ksi * kper, k1 = min(P.k, k0 + kper);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int slab = warp & 1, rq = warp >> 1;  // rows 16 slab .., ranks 16 rq ..
  const int lrow = tid >> 3, row = tile * kTRows + lrow;
  const int64_t xrow = row < P.rows ? (P.row_ids ? (int64_t)P.row_ids[row] : (int64_t)row) * P.ldx : int64_t(-1);
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  float xv[8], sv[8];
  uint4 cv;
  if (P.rchunks == 1)  // ranks past the rank stay 0 (the contiguous-run path writes only j < rank)
    for (int e = tid; e < (64 - P.rank) * 72; e += blockDim.x) sm.ct[P.rank + e / 72][e % 72] = __float2half_rn(0.0f);
  if (k0 < k1) t_tc_load(P, k0, ch, tid, xrow, xv, sv, cv);
  for (int kb = k0; kb < k1; kb += 64) {
    {  // registers -> shared: p = x s' as hi / lo; C^T
      uint32_t hv[4], lv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float p0 = xv[2 * i] * (sv[2 * i] * (2.0f / 7.0f)), p1 = xv[2 * i + 1] * (sv[2 * i + 1] * (2.0f / 7.0f));
        const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
        hv[i] = h2_as_u32(__halves2half2(h0, h1));
        lv[i] = h2_as_u32(__floats2half2_rn(p0 - __half2float(h0), p1 - __half2float(h1)));
      }
      const int k8 = (tid & 7) * 8;
      *reinterpret_cast<uint4*>(&sm.xh[lrow][k8]) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
      *reinterpret_cast<uint4*>(&sm.xl[lrow][k8]) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
      const uint32_t w[4] = {cv.x, cv.y, cv.z, cv.w};
      if (P.rchunks == 1) {  // byte e = 16 tid + i of the run: k row e / rank, rank e % rank
        const int e0 = 16 * tid;
        int kk = e0 / P.rank, j = e0 - kk * P.rank;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (kk < 64) sm.ct[j][kk] = __float2half_rn((float)((w[i >> 2] >> (8 * (i & 3))) & 0xFFu) - 4.0f);
          if (++j == P.rank) {
            j = 0;
            ++kk;
          }
        }
      } else {
        const int kk = tid >> 2, jl = (tid & 3) * 16;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          sm.ct[jl + i][kk] = __float2half_rn((float)((w[i >> 2] >> (8 * (i & 3))) & 0xFFu) - 4.0f);
      }
    }
    __syncthreads();
    if (kb + 64 < k1) t_tc_load(P, kb + 64, ch, tid, xrow, xv, sv, cv);  // next block in flight
#pragma unroll
    for (int k16 = 0; k16 < 4; ++k16) {
      const int kc = 16 * k16 + 2 * q, r0 = 16 * slab + g;
      uint32_t ah[4], al[4];
      ah[0] = *reinterpret_cast<const uint32_t*>(&sm.xh[r0][kc]);
      ah[1] = *reinterpret_cast<const uint32_t*>(&sm.xh[r0 + 8][kc]);
      ah[2] = *reinterpret_cast<const uint32_t*>(&sm.xh[r0][kc + 8]);
      ah[3] = *reinterpret_cast<const uint32_t*>(&sm.xh[r0 + 8][kc + 8]);
      al[0] = *reinterpret_cast<const uint32_t*>(&sm.xl[r0][kc]);
      al[1] = *reinterpret_cast<const uint32_t*>(&sm.xl[r0 + 8][kc]);
      al[2] = *reinterpret_cast<const uint32_t*>(&sm.xl[r0][kc + 8]);
      al[3] = *reinterpret_cast<const uint32_t*>(&sm.xl[r0 + 8][kc + 8]);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int n = 16 * rq + 8 * nt + g;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&sm.ct[n][kc]);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&sm.ct[n][kc + 8]);
        mma_16816(acc[nt], ah, b0, b1);
        mma_16816(acc[nt], al, b0, b1);
      }
    }
    __syncthreads();
  }
  const int r64 = P.rchunks * 64;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int col = ch * 64 + 16 * rq + 8 * nt + 2 * q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = tile * kTRows + 16 * slab + g + 8 * h;
      if (r < P.rows)
        *reinterpret_cast<float2*>(&P.part[((int64_t)ksi * P.rows + r) * r64 + col]) =
            make_float2(acc[nt][2 * h], acc[nt][2 * h + 1]);
    }
  }
}

// dev_counts (nullable): {n_probs, units} from moe_plan_kernel; the CTAs then
// loop over the planned units (grid-stride), else CTA = unit.  Symm-INT3
// factors take the tensor-core unit, real-valued ones the CUDA-core unit.
struct TCoreSmem {  // pf_t_unit's operands
  float sx[kTRows][68];  // rows 16 B aligned: float4 reads of 4 k
  float su[64][65];
};
// KIND 0: the units of symm-INT3 factors (tensor cores); KIND 1: real-valued
// factors (CUDA cores).  Launch both when a table mixes them.
template <int KIND>
__device__ __forceinline__ void pf_t_any_unit(const TProb* __restrict__ probs, int n_probs, int unit, uint8_t* sm) {
  int lo = 0, hi = n_probs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (probs[mid].unit0 <= unit) lo = mid; else hi = mid - 1;
  }
  if ((probs[lo].ucodes != nullptr) != (KIND == 0)) return;
  if (KIND == 0) {
    pf_t_tc_unit(probs[lo], unit - probs[lo].unit0, *reinterpret_cast<TTcSmem*>(sm));
  } else {
    TCoreSmem& c = *reinterpret_cast<TCoreSmem*>(sm);
    pf_t_unit(probs, n_probs, unit, c.sx, c.su);
  }
}
template <int KIND>
__global__ void __launch_bounds__(256, KIND == 0 ? 4 : 1) pf_t_kernel(const TProb* __restrict__ probs, int n_probs,
                                                                    const int32_t* __restrict__ dev_counts) {
  pdl_wait();  // inputs come from the preceding grid (programmatic dependent launch)
  constexpr int kSm = KIND == 0 ? sizeof(TTcSmem) : sizeof(TCoreSmem);
  __shared__ __align__(16) uint8_t sm[kSm];
  if (dev_counts == nullptr) {
    pf_t_any_unit<KIND>(probs, n_probs, blockIdx.x, sm);
    return;
  }
  n_probs = dev_counts[0];
  const int units = dev_counts[1];
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    pf_t_any_unit<KIND>(probs, n_probs, u, sm);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Grouped activation images + LoRC t partials, one launch per GEMM phase.
// CTA = (job, token tile, 64-k stage): the tile's rows (gathered, binary16)
// become the stage's SW128 image, and while they sit in shared memory the CTA
// also computes t = half(x) U over its 64 k for up to two compensators (fp32,
// the reference's Eigen product order-independent up to rounding), written as
// partials [k/64][rows][r64] that pf_t_images_kernel sums in stage order.
// ---------------------------------------------------------------------------
struct ImgT {
  const uint8_t* ucodes;  // k x rank symm-int3 codes (or null -> ureal)
  const float* uscales;   // k x gpr
  const float* ureal;     // k x rank
  int32_t rank, gpr, rchunks;
  float* part;            // [k/64][rows][rchunks * 64]
};
struct ImgJob {
  const void* x;
  int32_t x_dtype;
  int64_t ldx;
  const int32_t* row_ids;  // null: identity
  int32_t rows, k, ntok;
  uint8_t* img;            // [tok_tiles][k/64][ntok x 128 B]
  int32_t n_t;             // LoRC targets (0..2)
  ImgT t[2];
  int32_t blk0;            // first CTA of this job
};
constexpr int kImgTSmem = (kPfN * 65 + 64 * 65) * 4;

template <bool WITH_T>
__device__ __forceinline__ void pf_img_t_unit(const ImgJob* __restrict__ jobs, int n_jobs, int blk) {
  extern __shared__ float imgt_sm[];
  float* sx = imgt_sm;             // [ntok][65]
  float* su = imgt_sm + kPfN * 65; // [64][65]
  int lo = 0, hi = n_jobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].blk0 <= blk) lo = mid; else hi = mid - 1;
  }
  const ImgJob& J = jobs[lo];
  const int ks = J.k / kPfK;
  const int rel = blk - J.blk0;
  const int tile = rel / ks, st = rel % ks;
  const int ntok = J.ntok, tid = threadIdx.x;
  uint8_t* dst = J.img + (int64_t)rel * ntok * 128;
  for (int c = tid; c < ntok * 4; c += blockDim.x) {  // 16-k blocks
    const int r = c >> 2, b = c & 3;
    const int row = tile * ntok + r;
    uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if (row < J.rows)
      pf_load_block16(J.x, J.x_dtype, J.row_ids ? J.row_ids[row] : row, J.ldx, (int64_t)st * kPfK + b * 16, w);
    pf_store_block16(dst, r, b, w);
    if (WITH_T && J.n_t > 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float2 f = __half22float2(u32_as_h2(w[u]));
        sx[r * 65 + b * 16 + 2 * u] = f.x;
        sx[r * 65 + b * 16 + 2 * u + 1] = f.y;
      }
    }
  }
  if (!WITH_T || J.n_t == 0) return;
  const int j = tid & 63, rg = tid >> 6;  // rank column, row group (rows rg, rg + 4, ...)
  const int nr4 = ntok / 4;               // rows per thread (ntok is a multiple of 16)
  for (int ti = 0; ti < J.n_t; ++ti) {
    const ImgT& T = J.t[ti];
    const int r64 = T.rchunks * 64;
    for (int ch = 0; ch < T.rchunks; ++ch) {
      __syncthreads();  // sx written / su free
      for (int e = tid; e < 64 * 64; e += blockDim.x) {  // U tile [64 k][64 ranks] (lowrank.cpp:122-134)
        const int kk = e >> 6, jj = e & 63;
        const int kr = st * kPfK + kk, rc = ch * 64 + jj;
        float v = 0.0f;
        if (rc < T.rank) {
          if (T.ucodes) {
            const float sp = T.uscales[(int64_t)kr * T.gpr + rc / 64] * (2.0f / 7.0f);
            v = sp * ((float)T.ucodes[(int64_t)kr * T.rank + rc] - 4.0f);
          } else {
            v = T.ureal[(int64_t)kr * T.rank + rc];
          }
        }
        su[kk * 65 + jj] = v;
      }
      __syncthreads();
      float acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = 0.0f;
#pragma unroll 4
      for (int kk = 0; kk < 64; ++kk) {
        const float uv = su[kk * 65 + j];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nr4) acc[i] += sx[(rg + 4 * i) * 65 + kk] * uv;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int row = tile * ntok + rg + 4 * i;
        if (i < nr4 && row < J.rows) T.part[((int64_t)st * J.rows + row) * r64 + ch * 64 + j] = acc[i];
      }
    }
  }
}

// dev_counts (nullable): {n_jobs, blocks} written by moe_plan_kernel; the CTAs
// then loop over the planned blocks (grid-stride), else CTA = block.
// WITH_T = false: images only (the MoE prefill plan computes t separately) -- a
// small register footprint, so many CTAs per SM (the t variant holds ~170).
template <bool WITH_T>
__global__ void __launch_bounds__(256) pf_img_t_kernel(const ImgJob* __restrict__ jobs, int n_jobs,
                                                      const int32_t* __restrict__ dev_counts) {
  pdl_wait();  // inputs come from the preceding grid (programmatic dependent launch)
  if (dev_counts == nullptr) {
    pf_img_t_unit<WITH_T>(jobs, n_jobs, blockIdx.x);
    return;
  }
  n_jobs = dev_counts[0];
  const int blocks = dev_counts[1];
  for (int b = blockIdx.x; b < blocks; b += gridDim.x) {
    pf_img_t_unit<WITH_T>(jobs, n_jobs, b);
    __syncthreads();
  }
}

// Sums the k-split partials in split order and writes the hi / lo images.
__global__ void pf_t_images_kernel(const TProb* __restrict__ probs, int n_probs,
                                   const int32_t* __restrict__ dev_counts) {
  pdl_wait();  // inputs come from the preceding grid (programmatic dependent launch)
  if (dev_counts != nullptr) n_probs = dev_counts[0];
  for (int pi = blockIdx.y; pi < n_probs; pi += gridDim.y) {
  const TProb& P = probs[pi];
  const int r64 = P.rchunks * 64;
  const int ntok = P.ntok;
  const int tiles = (P.rows + ntok - 1) / ntok;
  const int total = tiles * ntok * r64;  // 32-bit index math (64-bit divisions are software routines)
  const int64_t sstride = (int64_t)P.rows * r64;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int row = (e >> 6) / P.rchunks, c = e - row * r64;
    float t = 0.0f;
    if (row < P.rows) {
      const float* pp = P.part + (int64_t)row * r64 + c;
#pragma unroll 4
      for (int s = 0; s < P.ks; ++s) t += pp[s * sstride];
    }
    const __half h = __float2half_rn(t);
    const __half l = __float2half_rn(t - __half2float(h));
    const int tile = row / ntok, r = row % ntok, ch = c / 64, jj = c % 64;
    const int ib = ntok * 128;
    uint8_t* base = P.timg + ((int64_t)(tile * P.rchunks + ch) * 2) * ib;
    const uint32_t off = (uint32_t)r * 128u + (uint32_t)(((jj >> 3) ^ (r & 7)) << 4) + (uint32_t)((jj & 7) * 2);
    *reinterpret_cast<__half*>(base + off) = h;
    *reinterpret_cast<__half*>(base + ib + off) = l;
  }
  }  // probs
}

}  // namespace milo_dev

namespace milo_dev {

// ---------------------------------------------------------------------------
// MoE prefill planned on the device (no host round trip: the whole layer call
// is stream-ordered and graph-capturable).  One CTA turns the routing ids into
// every table the prefill kernels read -- the reference composition order
// (SURVEY.md section 8b): per expert, its (token, k) entries in ascending token
// order, then the shared experts with every token -- and into the device-side
// counts the launches use (their grids are host bounds; CTAs past the planned
// work exit).  Workspace regions are sized on the host for the worst routing.
// ---------------------------------------------------------------------------
struct PfMatStatic {
  const uint8_t* w;        // macro tiles
  const uint8_t* vimg;     // V^T images (null: no LoRC)
  const uint8_t* ucodes;
  const float* uscales;
  const float* ureal;
  int32_t k, n, mode, rank, gpr, rch;
};
struct PfExpertStatic {
  PfMatStatic m[3];  // w1, w3, w2
};

// counts[] layout (int32): per phase ph (0, 1) at 16 * ph:
//   [0] n_jobs  [1] img blocks  [2] n_tprobs  [3] t units  [4] n_problems  [5] n_items  [6] ntok_max
struct PfPlanArgs {
  const int32_t* ids;             // m x K routing (-1 = unused)
  int32_t ids_cached;             // the ids fit the launch's dynamic shared memory (m K int32)
  int32_t ng2;                    // phase-2 (w2) items cover two 128-column n-tiles (pf_gemm_kernel<1, 2>)
  long long* dbg;                 // optional: globaltimer after each planning step (debug)
  int64_t m;
  int32_t K, E, S, sms;
  const PfExpertStatic* ex;       // E routed then S shared
  const void* x;
  int32_t x_dtype;
  int64_t d, f_max;
  // outputs
  int32_t* tok;                   // R grouped rows: x row
  int32_t* slot;                  // R grouped rows: Y slot
  ImgJob* jobs[2];                // <= G each
  TProb* tps[2];                  // <= 2G / G
  PfProblem* probs[2];            // <= G each
  int32_t* starts[2];             // G + 1 each
  int32_t* counts;                // 32 ints
  // regions (sized by the host for the worst case)
  uint8_t* img[2];                // activation images per phase
  uint8_t* timg[3];               // t images per matrix
  uint8_t* part[3];               // t partials per matrix
  __half* h;                      // R x f_max
  float* Y;                       // (m K + S m) x d
};

__device__ __forceinline__ int pf_ntok_dev(int64_t rows) { return (int)min((int64_t)kPfN, (rows + 15) / 16 * 16); }
__device__ __forceinline__ int pf_t_splits_dev(int rows, int k, int rch, int sms) {  // 32-bit: one thread per group
  const int row_tiles = (rows + kTRows - 1) / kTRows;
  return max(1, min(k / 256, (kTCtasPerSm * sms) / max(1, row_tiles * rch)));
}

constexpr int kPlanMaxGroups = 256;  // >= E + S (kRouteMaxE)
constexpr int kPlanIdsSmem = 160 * 1024;  // routing ids cached in shared memory up to this size

__global__ void __launch_bounds__(1024) moe_plan_kernel(PfPlanArgs a) {
  pdl_wait();  // inputs come from the preceding grid (programmatic dependent launch)
  auto stamp = [&](int i) {
    if (a.dbg != nullptr && threadIdx.x == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.dbg[i] = t;
    }
  };
  stamp(0);
  __shared__ int32_t s_cnt[kPlanMaxGroups];   // rows per expert (routed, shared)
  __shared__ int32_t s_off[kPlanMaxGroups];   // grouped row offset
  __shared__ int32_t s_gexp[kPlanMaxGroups];  // group -> expert
  __shared__ int32_t s_gofe[kPlanMaxGroups];  // expert -> group
  __shared__ int64_t s_o[8][kPlanMaxGroups];  // per group: img1, img2, timg0..2, part0..2 byte offsets
  __shared__ int32_t s_blk[2][kPlanMaxGroups], s_unit[3][kPlanMaxGroups], s_item[2][kPlanMaxGroups + 1];
  __shared__ int32_t s_ng;
  __shared__ int32_t s_shape[kPlanMaxGroups][3][4];  // per expert, matrix: k, n, rank, rch
  __shared__ int32_t s_tp[2][kPlanMaxGroups];        // per group: first t-problem slot per phase
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int E = a.E, S = a.S, K = a.K;
  const int64_t m = a.m, mK = m * K;
  // the routing ids in shared memory when they fit: the per-expert ballot scans
  // below read them E + S times (global round trips dominated the plan)
  extern __shared__ int32_t s_ids[];
  const int32_t* ids = a.ids;
  if (a.ids_cached) {
    for (int64_t i = tid; i < mK; i += blockDim.x) s_ids[i] = a.ids[i];
    ids = s_ids;
  }
  __syncthreads();
  for (int i = tid; i < (E + S) * 3; i += blockDim.x) {  // one parallel pass over the static table
    const PfMatStatic& M = a.ex[i / 3].m[i % 3];
    s_shape[i / 3][i % 3][0] = M.k;
    s_shape[i / 3][i % 3][1] = M.n;
    s_shape[i / 3][i % 3][2] = M.rank;
    s_shape[i / 3][i % 3][3] = M.rch;
  }
  stamp(1);
  // 1. rows per expert.  Cached ids: warp w counts the experts of its contiguous
  //    chunk of entries (__match_any_sync per 32-entry window) into hist[w][e],
  //    then thread e turns the counts into per-warp offsets (step 3 reuses them)
  //    and its total.  Otherwise one warp per expert scans every entry.
  const int n_ent = (int)mK;
  const int chunk = ((n_ent + nwarps * 32 - 1) / (nwarps * 32)) * 32;
  int32_t* hist = s_ids + ((n_ent + 3) & ~3);  // [nwarps][kPlanMaxGroups] (cached path)
  if (a.ids_cached) {
    for (int i = tid; i < nwarps * kPlanMaxGroups; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int b0 = warp * chunk, b1 = min(n_ent, b0 + chunk);
    for (int base = b0; base < b1; base += 32) {
      const int i = base + lane;
      const int e = i < b1 ? ids[i] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      if (e >= 0 && e < E && lane == __ffs(peers) - 1) hist[warp * kPlanMaxGroups + e] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    if (tid < E) {
      int run = 0;
      for (int w = 0; w < nwarps; ++w) {
        const int c = hist[w * kPlanMaxGroups + tid];
        hist[w * kPlanMaxGroups + tid] = run;
        run += c;
      }
      s_cnt[tid] = run;
    } else if (tid < E + S) {
      s_cnt[tid] = (int32_t)m;
    }
  }
  for (int e = warp; !a.ids_cached && e < E + S; e += nwarps) {
    int64_t c = 0;
    if (e < E) {
      const int n = (int)mK;
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool hit = i < n && ids[i] == e;
        c += __popc(__ballot_sync(0xffffffffu, hit));
      }
    } else {
      c = m;
    }
    if (lane == 0) s_cnt[e] = (int32_t)c;
  }
  __syncthreads();
  stamp(2);
  // 2. groups (non-empty experts, expert order) and every per-group offset: thread e
  //    sizes expert e's group, block-wide exclusive scans place them (a one-thread
  //    loop over the groups cost 70-100 us at 66-128 experts)
  {
    constexpr int kQ = 18;  // scanned quantities
    // 32-bit scans: byte offsets in 256-byte units (every region is 256-aligned)
    int32_t v[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) v[i] = 0;
    const int e = tid;
    const int rows = e < E + S ? s_cnt[e] : 0;
    const int nt = rows > 0 ? pf_ntok_dev(rows) : 0;
    const int tiles = rows > 0 ? (rows + nt - 1) / nt : 0;
    int ks_j[3] = {0, 0, 0};
    if (rows > 0) {
      v[0] = 1;     // group index
      v[1] = rows;  // grouped row offset
      // images: phase 1 over d, phase 2 over this expert's f (regions sized with f_max)
      v[2] = (int32_t)(((int64_t)tiles * (a.d / kPfK) * nt * 128 + 255) >> 8);
      v[3] = (int32_t)(((int64_t)tiles * (a.f_max / kPfK) * nt * 128 + 255) >> 8);
      v[4] = tiles * (int)(a.d / kPfK);
      v[5] = tiles * (s_shape[e][2][0] / kPfK);
      for (int j = 0; j < 3; ++j) {
        const int mk = s_shape[e][j][0], rank = s_shape[e][j][2], rch = s_shape[e][j][3];
        if (rank <= 0) continue;
        v[6 + j] = (int32_t)(((int64_t)tiles * rch * 2 * nt * 128 + 255) >> 8);
        const int ks = pf_t_splits_dev(rows, mk, rch, a.sms);
        ks_j[j] = ks;
        v[9 + j] = (int32_t)(((int64_t)max(mk / kPfK, ks) * rows * rch * 64 * 4 + 255) >> 8);
        v[12 + (j == 2 ? 1 : 0)] += ((rows + kTRows - 1) / kTRows) * rch * ks;  // t units per phase
        v[14 + (j == 2 ? 1 : 0)] += 1;                                                  // t problems per phase
      }
      v[16] = (s_shape[e][0][1] / kPfM) * tiles;
      v[17] = (s_shape[e][2][1] / (kPfM * (a.ng2 ? 2 : 1))) * tiles;
    }
    // warp inclusive scans, then the warps' totals
    __shared__ int32_t s_wtot[32][kQ];
    __shared__ int32_t s_ntmax;
    if (tid == 0) s_ntmax = 16;
    int32_t inc[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) {
      int32_t x = v[i];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      inc[i] = x;
      if (lane == 31) s_wtot[warp][i] = x;
    }
    __syncthreads();
    if (nt > 0) atomicMax(&s_ntmax, nt);
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < kQ; ++i) {
        const int32_t t = lane < nwarps ? s_wtot[lane][i] : 0;
        int32_t x = t;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        if (lane < nwarps) s_wtot[lane][i] = x - t;  // exclusive warp offsets
      }
    }
    __syncthreads();
    int32_t ex[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) ex[i] = s_wtot[warp][i] + inc[i] - v[i];
    if (rows > 0) {
      const int g = (int)ex[0];
      s_gexp[g] = e;
      s_gofe[e] = g;
      s_off[g] = (int32_t)ex[1];
      s_o[0][g] = (int64_t)ex[2] << 8;
      s_o[1][g] = (int64_t)ex[3] << 8;
      s_blk[0][g] = (int32_t)ex[4];
      s_blk[1][g] = (int32_t)ex[5];
      s_tp[0][g] = (int32_t)ex[14];
      s_tp[1][g] = (int32_t)ex[15];
      int32_t u01 = ex[12];  // w1 then w3 within the group (phase-wide prefix)
      for (int j = 0; j < 3; ++j) {
        s_o[2 + j][g] = (int64_t)ex[6 + j] << 8;
        s_o[5 + j][g] = (int64_t)ex[9 + j] << 8;
        s_unit[j][g] = 0;
        if (s_shape[e][j][2] <= 0) continue;
        const int32_t units = ((rows + kTRows - 1) / kTRows) * s_shape[e][j][3] * ks_j[j];
        if (j < 2) {
          s_unit[j][g] = (int32_t)u01;
          u01 += units;
        } else {
          s_unit[j][g] = (int32_t)ex[13];
        }
      }
      s_item[0][g] = (int32_t)ex[16];
      s_item[1][g] = (int32_t)ex[17];
    }
    if (tid == blockDim.x - 1) {  // totals: the last thread's inclusive values
      const int ng = (int)(ex[0] + v[0]);
      s_ng = ng;
      s_item[0][ng] = (int32_t)(ex[16] + v[16]);
      s_item[1][ng] = (int32_t)(ex[17] + v[17]);
    }
    __syncthreads();
    if (tid == blockDim.x - 1) {
      const int ng = s_ng;
      for (int ph = 0; ph < 2; ++ph) {
        int32_t* c = a.counts + 16 * ph;
        c[0] = ng;
        c[1] = (int32_t)(ex[4 + ph] + v[4 + ph]);
        c[2] = (int32_t)(ex[14 + ph] + v[14 + ph]);
        c[3] = (int32_t)(ex[12 + ph] + v[12 + ph]);
        c[4] = ng;
        c[5] = (int32_t)(ex[16 + ph] + v[16 + ph]);
        c[6] = s_ntmax;
      }
    }
  }
  __syncthreads();
  const int ng = s_ng;
  stamp(3);
  // 3. grouped rows: token (x row) and Y slot, entries of an expert in (t, k) order
  if (a.ids_cached) {  // the same windows as step 1: offset = group + earlier warps + rank in the window
    const int b0 = warp * chunk, b1 = min(n_ent, b0 + chunk);
    for (int base = b0; base < b1; base += 32) {
      const int i = base + lane;
      const int e = i < b1 ? ids[i] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      if (e >= 0 && e < E) {
        int32_t* h = hist + warp * kPlanMaxGroups + e;
        const int p = s_off[s_gofe[e]] + *h + __popc(peers & ((1u << lane) - 1u));
        a.tok[p] = i / K;
        a.slot[p] = i;
      }
      __syncwarp();
      if (e >= 0 && e < E && lane == __ffs(peers) - 1) hist[warp * kPlanMaxGroups + e] += __popc(peers);
      __syncwarp();
    }
  }
  for (int g = warp; g < ng; g += nwarps) {
    const int e = s_gexp[g];
    int32_t* tok = a.tok + s_off[g];
    int32_t* slot = a.slot + s_off[g];
    if (e < E && a.ids_cached) continue;  // done above
    if (e < E) {  // (32-bit indices: mK < 2^31; a 64-bit division per hit cost ~10 us)
      const int n = (int)mK;
      int pos = 0;
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool hit = i < n && ids[i] == e;
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int p = pos + __popc(b & ((1u << lane) - 1u));
          tok[p] = i / K;
          slot[p] = i;
        }
        pos += __popc(b);
      }
    } else {
      for (int64_t t = lane; t < m; t += 32) {
        tok[t] = (int32_t)t;
        slot[t] = (int32_t)(mK + (int64_t)(e - E) * m + t);
      }
    }
  }
  __syncthreads();
  stamp(4);
  // 4. per-group tables (thread per group)
  for (int g = tid; g < ng; g += blockDim.x) {
    const int e = s_gexp[g];
    const PfExpertStatic& X = a.ex[e];
    const int64_t rows = s_cnt[e], off = s_off[g];
    const int nt = pf_ntok_dev(rows);
    // activation image jobs (no fused t: pf_t_kernel computes t)
    ImgJob J1{};
    J1.x = a.x;
    J1.x_dtype = a.x_dtype;
    J1.ldx = a.d;
    J1.row_ids = a.tok + off;
    J1.rows = (int32_t)rows;
    J1.k = (int32_t)a.d;
    J1.ntok = nt;
    J1.img = a.img[0] + s_o[0][g];
    J1.blk0 = s_blk[0][g];
    a.jobs[0][g] = J1;
    ImgJob J2{};
    J2.x = a.h + off * a.f_max;
    J2.x_dtype = 1;
    J2.ldx = a.f_max;
    J2.row_ids = nullptr;
    J2.rows = (int32_t)rows;
    J2.k = X.m[2].k;
    J2.ntok = nt;
    J2.img = a.img[1] + s_o[1][g];
    J2.blk0 = s_blk[1][g];
    a.jobs[1][g] = J2;
    // t problems: phase 1 in (group, w1, w3) order, phase 2 per group; the slot
    // of a group's problem is its rank among the groups before it with a comp
    int n0 = s_tp[0][g], n1 = s_tp[1][g];
    for (int j = 0; j < 3; ++j) {
      const PfMatStatic& M = X.m[j];
      if (M.rank <= 0) continue;
      TProb tp{};
      if (j < 2) {
        tp.x = a.x;
        tp.x_dtype = a.x_dtype;
        tp.ldx = a.d;
        tp.row_ids = a.tok + off;
      } else {
        tp.x = a.h + off * a.f_max;
        tp.x_dtype = 1;
        tp.ldx = a.f_max;
        tp.row_ids = nullptr;
      }
      tp.rows = (int32_t)rows;
      tp.k = M.k;
      tp.rank = M.rank;
      tp.gpr = M.gpr;
      tp.rchunks = M.rch;
      tp.ks = pf_t_splits_dev(rows, M.k, M.rch, a.sms);
      tp.ucodes = M.ucodes;
      tp.uscales = M.uscales;
      tp.ureal = M.ureal;
      tp.timg = a.timg[j] + s_o[2 + j][g];
      tp.part = reinterpret_cast<float*>(a.part[j] + s_o[5 + j][g]);
      tp.ntok = nt;
      tp.unit0 = s_unit[j][g];
      if (j < 2)
        a.tps[0][n0++] = tp;
      else
        a.tps[1][n1++] = tp;
    }
    // GEMM problems
    PfProblem P1{};
    P1.w[0] = X.m[0].w;
    P1.w[1] = X.m[1].w;
    P1.act = J1.img;
    for (int j = 0; j < 2; ++j)
      if (X.m[j].rank > 0) {
        P1.vimg[j] = X.m[j].vimg;
        P1.timg[j] = a.timg[j] + s_o[2 + j][g];
        P1.rchunks[j] = X.m[j].rch;
      }
    P1.k = (int32_t)a.d;
    P1.n = X.m[0].n;
    P1.rows = (int32_t)rows;
    P1.ntok = nt;
    P1.mode = X.m[0].mode;
    P1.kind = 1;
    P1.out_dtype = 1;
    P1.ldo = a.f_max;
    P1.out = a.h + off * a.f_max;
    a.probs[0][g] = P1;
    PfProblem P2{};
    P2.w[0] = X.m[2].w;
    P2.act = J2.img;
    if (X.m[2].rank > 0) {
      P2.vimg[0] = X.m[2].vimg;
      P2.timg[0] = a.timg[2] + s_o[4][g];
      P2.rchunks[0] = X.m[2].rch;
    }
    P2.k = X.m[2].k;
    P2.n = (int32_t)a.d;
    P2.rows = (int32_t)rows;
    P2.ntok = nt;
    P2.mode = X.m[2].mode;
    P2.kind = 0;
    P2.out_dtype = 0;
    P2.ldo = a.d;
    P2.out = a.Y;
    P2.row_map = a.slot + off;
    a.probs[1][g] = P2;
    a.starts[0][g] = s_item[0][g];
    a.starts[1][g] = s_item[1][g];
  }
  if (tid == 0) {
    a.starts[0][ng] = s_item[0][ng];
    a.starts[1][ng] = s_item[1][ng];
  }
  __syncthreads();
  stamp(5);
}

}  // namespace milo_dev
