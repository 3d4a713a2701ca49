// K3: the prefill-regime W3A16 + LoRC GEMM on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM), for token counts where the weights are
// worth reusing across many tokens (m_e >= ~64 per matrix).
//
// Reference semantics, per matrix: milo::gemm_w3a16 (proj/src/gemm.cpp:117-199)
//   C = half(A) * dequant(W) + (half(A) U) V, fp32 accumulation.
//
// Per work item (problem p, n-tile of 128 output columns = 2 slabs, token tile
// of 128 rows) one CTA computes D[128 n][128 tok] = W^T X^T in TMEM:
//   * producer warp : cp.async.bulk of the packed INT3 macro tiles (2 slabs x
//                     2 k-tiles per 64-k stage) and of the stage's activation
//                     "image" (16 KB, already binary16, SW128 K-major, built by
//                     pf_image_kernel), and of the LoRC images;
//   * dequant warps : packed tiles -> bit-exact binary16 weights written into
//                     the A operand (128 n rows x 64 k, SW128 K-major);
//   * MMA thread    : 4 x tcgen05.mma.kind::f16 (K = 16) per stage, then
//                     tcgen05.commit to release the stage;
//   * epilogue warps: tcgen05.ld (32 lanes x 32 columns) -> C rows / SwiGLU.
// The compensator term (t V) runs as extra K stages of the same accumulator:
// A = V^T image (hi or lo binary16 half of the fp32 values), B = t image (hi
// or lo), three MMAs per 64-rank chunk (hi.hi + hi.lo + lo.hi), i.e. fp32-level
// accuracy on the tensor cores.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "layout.cuh"
#include "ptx.cuh"

namespace milo_dev {

#ifndef PF_NG2_AS
#define PF_NG2_AS 3
#endif
#ifndef PF_NG2_GROUPS
#define PF_NG2_GROUPS 3
#endif
#ifndef PF_NG2_PS
#define PF_NG2_PS 6
#endif
#ifndef PF_NG2_B
#define PF_NG2_B 64
#endif
constexpr int kPfM = 128;              // output columns per tile (UMMA M)
constexpr int kPfN = 128;              // tokens per tile (UMMA N, TMEM columns)
constexpr int kPfK = 64;               // k per stage (128 B of binary16 per operand row)
constexpr int kPfImg = kPfN * kPfK * 2;  // 16 KB: one operand image (128 rows x 128 B)
constexpr int kPfPackedPerMat = 2 * 2 * kTileBytes;  // 2 slabs x 2 k-tiles = 3584 B
constexpr int kPfGroupWarps = 4;       // warps per dequant group (one group per in-flight stage)
constexpr int kPfEpiWarps = 4;         // warps 0..3: TMEM lanes 32 w .. 32 w + 31
constexpr int kPfProdWarp = 4;         // packed-weight producer
constexpr int kPfMmaWarp = 5;
constexpr int kPfBWarp = 6;            // activation / t image producer
constexpr int kPfDeqWarp0 = 7;
// NG = n-tiles (128 output columns each) per work item: the item's activation
// image of a stage feeds NG MMAs (NG accumulators), so activation traffic per
// FLOP drops by NG -- the activation ring, not the tensor core, bounds the
// NG = 1 kernel (one 16 KB image per 128 x 128 x 64 MMA, ~2 us copy latency).
// Groups <= A-ring slots: a group that starts stage st has only seen stage
// st - groups consumed, and its parity wait on the slot is unambiguous only
// if the slot's barrier is at most one phase behind (st - 2 AS consumed).
template <int NMAT, int NG = 1>
struct PfRoles {
  static constexpr int kGroups = NG == 2 ? PF_NG2_GROUPS : (NMAT == 1 ? 4 : 3);  // stages de-quantized concurrently
  static constexpr int kDeqWarps = kGroups * kPfGroupWarps;
  static constexpr int kThreads = 32 * (kPfDeqWarp0 + kDeqWarps);
};

template <int NMAT, int NG = 1>
struct PfCfg {
  // NG = 2: the packed (HBM) and activation (L2) rings are latency x depth
  // bound per SM, so they get the space and A keeps PF_NG2_AS slots
  static constexpr int kPS = NG == 2 ? PF_NG2_PS : (NMAT == 1 ? 12 : 8);      // packed-weight ring (HBM latency)
  static constexpr int kAS = NG == 2 ? PF_NG2_AS : (NMAT == 1 ? 6 : 3);       // dequantized A ring
  static constexpr int kBRegion = NG == 2 ? PF_NG2_B * 1024 : (NMAT == 1 ? 64 * 1024 : 32 * 1024);
  static constexpr int kBSMax = 16;                      // B slots = region / (ntok_max x 128), <= 16
  static constexpr int kStageA = NG * NMAT * kPfImg;
  static constexpr int kStageP = NG * NMAT * kPfPackedPerMat;
  static constexpr int kOffA = 0;                        // 1024-aligned images first
  static constexpr int kOffB = kOffA + kAS * kStageA;
  static constexpr int kOffP = kOffB + kBRegion;
  static constexpr int kOffBar = kOffP + kPS * kStageP;
  // p_full[PS] p_empty[PS] a_full[AS] a_empty[AS] v_full[AS] b_full[BSMax] b_empty[BSMax] acc_full[2] acc_empty[2]
  static constexpr int kNumBars = 2 * kPS + 3 * kAS + 2 * kBSMax + 4;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kOffStage = (kOffTmem + 16 + 127) & ~127;  // epilogue transpose [4 warps][32][33] f32
  static constexpr int kBytes = kOffStage + kPfEpiWarps * 32 * 33 * 4 + 1024;  // + alignment slack
  static constexpr int kTmemCols = 2 * NG * NMAT * kPfN;  // double-buffered accumulators
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
__device__ __forceinline__ void pf_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
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

// ---------------------------------------------------------------- the kernel
// Persistent: CTA c handles items c, c + grid, ...  Three rings decouple the
// roles: packed weights (deep, HBM latency), dequantized A, activation images.
// Every role walks the same stage sequence: per item, k / 64 main stages then
// 3 LoRC stages per 64-rank chunk per matrix.
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
  static_assert(kPfDeqGroups <= PfCfg<NMAT, NG>::kAS, "dequant groups must not outnumber A slots");
  using CF = PfCfg<NMAT, NG>;
  constexpr int PS = CF::kPS, AS = CF::kAS;
  const int bslot = a.ntok_max * 128;
  const int BS = min(CF::kBSMax, CF::kBRegion / bslot);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned base (SW128 atoms); pointer arithmetic keeps the shared address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::kOffBar);
  uint64_t* p_full = bars;
  uint64_t* p_empty = p_full + PS;
  uint64_t* a_full = p_empty + PS;
  uint64_t* a_empty = a_full + AS;
  uint64_t* v_full = a_empty + AS;
  uint64_t* b_full = v_full + AS;
  uint64_t* b_empty = b_full + CF::kBSMax;
  uint64_t* acc_full = b_empty + CF::kBSMax;  // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + CF::kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < PS; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&p_empty[s], kPfGroupWarps);
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(&a_full[s], kPfGroupWarps);
      mbar_init(&a_empty[s], 1);
      mbar_init(&v_full[s], 1);
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kPfEpiWarps);
    }
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
  auto pf_trace = [&](int stage, int role) {  // CTA 0, first 64 stages: [stage][4 roles]
    if (a.dbg != nullptr && blockIdx.x == 0 && stage < 64) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.dbg[148 * 8 + stage * 4 + role] = t;
    }
  };

  auto item_stages = [&](const PfProblem& P) {
    return P.k / kPfK + 3 * (P.rchunks[0] + (NMAT == 2 ? P.rchunks[1] : 0));
  };
  // LoRC stage l (0-based after the main stages) -> matrix, chunk, V part, t part
  auto lorc_stage = [&](const PfProblem& P, int l, int& mat, int& ch, int& vpart, int& tpart) {
    mat = 0;
    if (l >= 3 * P.rchunks[0]) {
      l -= 3 * P.rchunks[0];
      mat = 1;
    }
    ch = l / 3;
    const int part = l % 3;  // 0: V_hi.t_hi, 1: V_hi.t_lo, 2: V_lo.t_hi
    vpart = part == 2 ? 1 : 0;
    tpart = part == 1 ? 1 : 0;
  };

  if (warp == kPfProdWarp) {
    // ======================= packed-weight producer =======================
    // A stage's NG x NMAT x 2 copies are issued by as many lanes in parallel: one
    // thread serialises its bulk copies at ~300 cycles each (tools/micro/bulk_issue.cu).
    constexpr int kCopies = NG * NMAT * 2;
    if (lane < kCopies) {
      const int ng = lane / (NMAT * 2), mat = (lane / 2) % NMAT, sl = lane & 1;
      int ps = 0;
      uint32_t pph = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        int p, nt, tt;
        pf_item<NG>(a, item, p, nt, tt);
        const PfProblem P = a.problems[p];  // by value: fields live in registers
        const int ks = P.k / kPfK, kts = P.k / kTileK;
        for (int st = 0; st < ks; ++st) {
          ring_wait(&p_empty[ps], pph ^ 1);

          uint8_t* sP = smem + CF::kOffP + ps * CF::kStageP;
          if (lane == 0) mbar_arrive_expect_tx(&p_full[ps], (uint32_t)CF::kStageP);
          __syncwarp((1u << kCopies) - 1u);
          const int kst = (st + nt * 13) % ks;  // rotated k order per n-tile (spreads L2 hot spots)
          const uint8_t* src = P.w[mat] + ((int64_t)(2 * (NG * nt + ng) + sl) * kts + 2 * kst) * kTileBytes;
          bulk_g2s(sP + ((ng * NMAT + mat) * 2 + sl) * 2 * kTileBytes, src, 2 * kTileBytes, &p_full[ps]);
          if (item == (int)blockIdx.x && lane == 0) pf_trace(st, 0);

          if (++ps == PS) {
            ps = 0;
            pph ^= 1;
          }
        }
      }
      if (lane == 0) pf_dbg(1);
    }
  } else if (warp == kPfBWarp) {
    // ======================= activation / t image producer =======================
    if (lane == 0) {
      int bs = 0;
      uint32_t bph = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        int p, nt, tt;
        pf_item<NG>(a, item, p, nt, tt);
        const PfProblem P = a.problems[p];  // by value: fields live in registers
        const int ks = P.k / kPfK, total = item_stages(P);
        for (int st = 0; st < total; ++st) {
          ring_wait(&b_empty[bs], bph ^ 1);
          uint8_t* sB = smem + CF::kOffB + bs * bslot;
          const uint8_t* src;
          const uint32_t ib = (uint32_t)P.ntok * 128u;  // one token-tile image
          if (st < ks) {
            src = P.act + ((int64_t)tt * ks + (st + nt * 13) % ks) * ib;  // same rotation as the weights
          } else {
            int mat, ch, vpart, tpart;
            lorc_stage(P, st - ks, mat, ch, vpart, tpart);
            src = P.timg[mat] + (((int64_t)tt * P.rchunks[mat] + ch) * 2 + tpart) * ib;
          }
          mbar_arrive_expect_tx(&b_full[bs], ib);
          bulk_g2s(sB, src, ib, &b_full[bs]);
          if (item == (int)blockIdx.x) pf_trace(st, 3);
          if (++bs == BS) {
            bs = 0;
            bph ^= 1;
          }
        }
      }
      pf_dbg(2);
    }
  } else if (warp >= kPfDeqWarp0) {
    // ======================= dequant warps =======================
    // group grp handles the stages st = grp (mod kPfDeqGroups): two stages are
    // de-quantized concurrently; within a stage, warp gw does jobs gw, gw + 4, ...
    const int dw = warp - kPfDeqWarp0;
    const int grp = dw / kPfGroupWarps, gw = dw % kPfGroupWarps;
    const int g = lane >> 2, q = lane & 3;
    int ps = 0, as = 0, gs = 0;
    uint32_t pph = 0, aph = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      int p, nt, tt;
      pf_item<NG>(a, item, p, nt, tt);
      const PfProblem P = a.problems[p];  // by value: fields live in registers
      const int ks = P.k / kPfK, total = item_stages(P);
      const DqConsts dq = make_dq_consts(P.mode);
      for (int st = 0; st < total; ++st, ++gs) {
        const bool mine = (gs % kPfDeqGroups) == grp;
        uint8_t* sA = smem + CF::kOffA + as * CF::kStageA;
        if (mine) {
          // every warp of the group waits for the A slot (a parity wait on v_full
          // alone would pass early when this group's first stage reuses a slot
          // whose previous phase has not completed yet); the first warp then
          // either fetches a V image into it (LoRC stage) or releases v_full
          ring_wait(&a_empty[as], aph ^ 1);
          if (gw == 0 && lane == 0) {
            if (st >= ks) {
              int mat, ch, vpart, tpart;
              lorc_stage(P, st - ks, mat, ch, vpart, tpart);
              mbar_arrive_expect_tx(&v_full[as], (uint32_t)(NG * kPfImg));
              for (int ng = 0; ng < NG; ++ng)
                bulk_g2s(sA + (ng * NMAT + mat) * kPfImg,
                         P.vimg[mat] + (((int64_t)(NG * nt + ng) * P.rchunks[mat] + ch) * 2 + vpart) * kPfImg, kPfImg,
                         &v_full[as]);
            } else {
              mbar_arrive(&v_full[as]);
            }
          }
          ring_wait(&v_full[as], aph);
          if (st < ks) {
            ring_wait(&p_full[ps], pph);
            if (gw == 0 && lane == 0 && item == (int)blockIdx.x) pf_trace(st, 1);
            const uint8_t* sP = smem + CF::kOffP + ps * CF::kStageP;
            constexpr int kJobs = 8 * NMAT * NG / kPfGroupWarps;
#pragma unroll
            for (int jb = 0; jb < ((a.flags & 1) ? 0 : kJobs); ++jb) {
              const int jid = gw + kPfGroupWarps * jb;
              const int j = jid & 1, t4 = jid >> 1;
              const int kt = t4 & 1, sl = (t4 >> 1) & 1, nm = t4 >> 2;  // nm = ng * NMAT + mat
              const uint8_t* tile = sP + ((nm * 2 + sl) * 2 + kt) * kTileBytes;
              const uint32_t* pa = reinterpret_cast<const uint32_t*>(tile + kPlaneAOff + lane * 16);
              const uint32_t* pb = reinterpret_cast<const uint32_t*>(tile + kPlaneBOff + lane * 8);
              const uint4 mm = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32 + 16 * j);
              const uint32_t S2[2] = {mm.x, mm.z}, O2[2] = {mm.y, mm.w};
              uint32_t wv[16];
              unit_dequant(pa[2 * j], pa[2 * j + 1], pb[j], S2, O2, dq, wv);
              uint8_t* A = sA + nm * kPfImg;
#pragma unroll
              for (int pp = 0; pp < 16; ++pp) {
                const int i = pp >> 2, r = pp & 3;
                const int n = sl * 64 + 16 * i + g + 8 * (r & 1);
                const int k = kt * 32 + 16 * j + 2 * q + 8 * (r >> 1);
                const uint32_t off = (uint32_t)n * 128u + (uint32_t)(((k >> 3) ^ (n & 7)) << 4) + (uint32_t)((k & 7) * 2);
                *reinterpret_cast<uint32_t*>(A + off) = wv[pp];
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_empty[ps]);
            if (!(a.flags & 16)) fence_proxy_async();  // generic smem writes -> tensor-core (async proxy) reads
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_full[as]);

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
    if (dw == 0 && lane == 0) pf_dbg(3);
  } else if (warp == kPfMmaWarp) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        int p, nt, tt;
        pf_item<NG>(a, item, p, nt, tt);
        const PfProblem P = a.problems[p];  // by value: fields live in registers
        const int ks = P.k / kPfK, total = item_stages(P);
        const uint32_t idesc = pf_idesc(P.ntok);
        ring_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + (uint32_t)(acc * NG * NMAT * kPfN);
        for (int st = 0; st < total; ++st) {
          ring_wait(&a_full[as], aph);

          ring_wait(&b_full[bs], bph);
          tc_fence_after();
          const uint32_t aA = smem_u32(smem + CF::kOffA + as * CF::kStageA);
          const uint32_t aB = smem_u32(smem + CF::kOffB + bs * bslot);
          int mat0 = 0, mat1 = NMAT;
          if (st >= ks) {
            int mat, ch, vpart, tpart;
            lorc_stage(P, st - ks, mat, ch, vpart, tpart);
            mat0 = mat;
            mat1 = mat + 1;
          }
          for (int ng = 0; ng < NG; ++ng)
            for (int mat = mat0; mat < mat1; ++mat) {
#pragma unroll
              for (int k16 = 0; k16 < kPfK / 16; ++k16) {
                const uint64_t da = pf_desc_sw128(aA + (ng * NMAT + mat) * kPfImg + k16 * 32);
                const uint64_t db = pf_desc_sw128(aB + k16 * 32);
                if (!(a.flags & 2))
                  pf_mma(d0 + (uint32_t)((ng * NMAT + mat) * kPfN), da, db, idesc, (st > 0 || k16 > 0) ? 1u : 0u);
              }
            }
          pf_commit(&a_empty[as]);
          pf_commit(&b_empty[bs]);
          if ((a.flags & 32) && item == (int)blockIdx.x && st < 64) {  // debug: commit latency
            pf_trace(st, 1);
            ring_wait(&a_empty[as], aph);
            pf_trace(st, 3);
          }
          if (item == (int)blockIdx.x) pf_trace(st, 2);
          if (++as == AS) {
            as = 0;
            aph ^= 1;
          }
          if (++bs == BS) {
            bs = 0;
            bph ^= 1;
          }
        }
        pf_commit(&acc_full[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      pf_dbg(4);
    }
  } else {
    // ======================= epilogue warps 0..3 =======================
    const int ew = warp;  // TMEM lanes 32 ew .. 32 ew + 31 = A rows (output columns)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      int p, nt, tt;
      pf_item<NG>(a, item, p, nt, tt);
      const PfProblem P = a.problems[p];  // by value: fields live in registers
      ring_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      if (threadIdx.x == 0) pf_dbg(6);
      // TMEM -> registers (thread = output column, 32 tokens per load) -> SwiGLU /
      // identity -> smem transpose -> 16-byte row stores (8 token rows per instruction)
      const int rows = P.rows, kind = P.kind, odt = P.out_dtype;
      const int64_t ldo = P.ldo;
      const int32_t* rmap = P.row_map;
      float* stg = reinterpret_cast<float*>(smem + CF::kOffStage) + ew * 32 * 33;
      const int ntok = P.ntok;
#pragma unroll 1
      for (int ng = 0; ng < NG; ++ng) {
      const uint32_t tbase = tmem + ((uint32_t)(32 * ew) << 16) + (uint32_t)((acc * NG + ng) * NMAT * kPfN);
      const int col0 = (NG * nt + ng) * kPfM + 32 * ew + 8 * (lane & 3);  // this lane's 8 output columns
#pragma unroll 1
      for (int c0 = 0; c0 < ntok; c0 += 32) {
        uint32_t v0[32], v1[32];
        tmem_ld32(tbase + (uint32_t)c0, v0);
        if (NMAT == 2) tmem_ld32(tbase + (uint32_t)(kPfN + c0), v1);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          float x = __uint_as_float(v0[c]);
          if (kind == 1) x = pf_silu(x) * (NMAT == 2 ? __uint_as_float(v1[c]) : 0.0f);
          stg[c * 33 + lane] = x;
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
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
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
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
__global__ void pf_image_kernel(const void* __restrict__ x, int32_t x_dtype, int64_t ldx,
                                const int32_t* __restrict__ row_ids, int32_t rows, int32_t k, int32_t ntok,
                                uint8_t* __restrict__ img) {
  const int ks = k / kPfK;
  const int tile = blockIdx.x / ks, st = blockIdx.x % ks;
  uint8_t* dst = img + (int64_t)blockIdx.x * ntok * 128;
  for (int c = threadIdx.x; c < ntok * 8; c += blockDim.x) {  // 16-B chunks
    const int r = c >> 3, ch = c & 7;
    const int row = tile * ntok + r;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (row < rows) {
      const int64_t src_row = row_ids ? row_ids[row] : row;
      const int64_t col = (int64_t)st * kPfK + ch * 8;
      if (x_dtype == 0) {
        const float4* s = reinterpret_cast<const float4*>(static_cast<const float*>(x) + src_row * ldx + col);
        const float4 p0 = s[0], p1 = s[1];
        v = make_uint4(h2_as_u32(__floats2half2_rn(p0.x, p0.y)), h2_as_u32(__floats2half2_rn(p0.z, p0.w)),
                       h2_as_u32(__floats2half2_rn(p1.x, p1.y)), h2_as_u32(__floats2half2_rn(p1.z, p1.w)));
      } else {
        v = *reinterpret_cast<const uint4*>(static_cast<const __half*>(x) + src_row * ldx + col);
      }
    }
    *reinterpret_cast<uint4*>(dst + r * 128 + ((ch ^ (r & 7)) << 4)) = v;
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
#define PF_T_CTAS 1
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

// dev_counts (nullable): {n_probs, units} from moe_plan_kernel; the CTAs then
// loop over the planned units (grid-stride), else CTA = unit.
__global__ void __launch_bounds__(256) pf_t_kernel(const TProb* __restrict__ probs, int n_probs,
                                                  const int32_t* __restrict__ dev_counts) {
  __shared__ __align__(16) float sx[kTRows][68];  // rows 16 B aligned: float4 reads of 4 k
  __shared__ float su[64][65];
  if (dev_counts == nullptr) {
    pf_t_unit(probs, n_probs, blockIdx.x, sx, su);
    return;
  }
  n_probs = dev_counts[0];
  const int units = dev_counts[1];
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    pf_t_unit(probs, n_probs, u, sx, su);
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
  for (int c = tid; c < ntok * 8; c += blockDim.x) {  // 16-B chunks
    const int r = c >> 3, ch = c & 7;
    const int row = tile * ntok + r;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (row < J.rows) {
      const int64_t src_row = J.row_ids ? J.row_ids[row] : row;
      const int64_t col = (int64_t)st * kPfK + ch * 8;
      if (J.x_dtype == 0) {
        const float4* sp = reinterpret_cast<const float4*>(static_cast<const float*>(J.x) + src_row * J.ldx + col);
        const float4 p0 = sp[0], p1 = sp[1];
        v = make_uint4(h2_as_u32(__floats2half2_rn(p0.x, p0.y)), h2_as_u32(__floats2half2_rn(p0.z, p0.w)),
                       h2_as_u32(__floats2half2_rn(p1.x, p1.y)), h2_as_u32(__floats2half2_rn(p1.z, p1.w)));
      } else {
        v = *reinterpret_cast<const uint4*>(static_cast<const __half*>(J.x) + src_row * J.ldx + col);
      }
    }
    *reinterpret_cast<uint4*>(dst + r * 128 + ((ch ^ (r & 7)) << 4)) = v;
    if (J.n_t > 0) {
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f = __half22float2(u32_as_h2(w[u]));
        sx[r * 65 + ch * 8 + 2 * u] = f.x;
        sx[r * 65 + ch * 8 + 2 * u + 1] = f.y;
      }
    }
  }
  if (J.n_t == 0) return;
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
__global__ void __launch_bounds__(256) pf_img_t_kernel(const ImgJob* __restrict__ jobs, int n_jobs,
                                                      const int32_t* __restrict__ dev_counts) {
  if (dev_counts == nullptr) {
    pf_img_t_unit(jobs, n_jobs, blockIdx.x);
    return;
  }
  n_jobs = dev_counts[0];
  const int blocks = dev_counts[1];
  for (int b = blockIdx.x; b < blocks; b += gridDim.x) {
    pf_img_t_unit(jobs, n_jobs, b);
    __syncthreads();
  }
}

// Sums the k-split partials in split order and writes the hi / lo images.
__global__ void pf_t_images_kernel(const TProb* __restrict__ probs, int n_probs,
                                   const int32_t* __restrict__ dev_counts) {
  if (dev_counts != nullptr) n_probs = dev_counts[0];
  for (int pi = blockIdx.y; pi < n_probs; pi += gridDim.y) {
  const TProb& P = probs[pi];
  const int r64 = P.rchunks * 64;
  const int ntok = P.ntok;
  const int tiles = (P.rows + ntok - 1) / ntok;
  const int64_t total = (int64_t)tiles * ntok * r64;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / r64), c = (int)(e % r64);
    float t = 0.0f;
    if (row < P.rows)
      for (int s = 0; s < P.ks; ++s) t += P.part[((int64_t)s * P.rows + row) * r64 + c];
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
__device__ __forceinline__ int pf_t_splits_dev(int64_t rows, int64_t k, int rch, int sms) {
  const int row_tiles = (int)((rows + kTRows - 1) / kTRows);
  return max(1, min((int)(k / 256), (kTCtasPerSm * sms) / max(1, row_tiles * rch)));
}

constexpr int kPlanMaxGroups = 256;  // >= E + S (kRouteMaxE)

__global__ void __launch_bounds__(1024) moe_plan_kernel(PfPlanArgs a) {
  __shared__ int32_t s_cnt[kPlanMaxGroups];   // rows per expert (routed, shared)
  __shared__ int32_t s_off[kPlanMaxGroups];   // grouped row offset
  __shared__ int32_t s_gexp[kPlanMaxGroups];  // group -> expert
  __shared__ int64_t s_o[8][kPlanMaxGroups];  // per group: img1, img2, timg0..2, part0..2 byte offsets
  __shared__ int32_t s_blk[2][kPlanMaxGroups], s_unit[3][kPlanMaxGroups], s_item[2][kPlanMaxGroups + 1];
  __shared__ int32_t s_ng;
  __shared__ int32_t s_shape[kPlanMaxGroups][3][4];  // per expert, matrix: k, n, rank, rch
  __shared__ int32_t s_tp[2][kPlanMaxGroups];        // per group: first t-problem slot per phase
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int E = a.E, S = a.S, K = a.K;
  const int64_t m = a.m, mK = m * K;
  for (int i = tid; i < (E + S) * 3; i += blockDim.x) {  // one parallel pass over the static table
    const PfMatStatic& M = a.ex[i / 3].m[i % 3];
    s_shape[i / 3][i % 3][0] = M.k;
    s_shape[i / 3][i % 3][1] = M.n;
    s_shape[i / 3][i % 3][2] = M.rank;
    s_shape[i / 3][i % 3][3] = M.rch;
  }
  // 1. rows per expert: one warp per expert scans the entries with ballots
  for (int e = warp; e < E + S; e += nwarps) {
    int64_t c = 0;
    if (e < E) {
      for (int64_t base = 0; base < mK; base += 32) {
        const int64_t i = base + lane;
        const bool hit = i < mK && a.ids[i] == e;
        c += __popc(__ballot_sync(0xffffffffu, hit));
      }
    } else {
      c = m;
    }
    if (lane == 0) s_cnt[e] = (int32_t)c;
  }
  __syncthreads();
  // 2. groups (non-empty experts, expert order) and every per-group offset (serial: <= 512 groups)
  if (tid == 0) {
    int ng = 0;
    int64_t off = 0, oimg[2] = {0, 0}, ot[3] = {0, 0, 0}, op[3] = {0, 0, 0};
    int32_t blk[2] = {0, 0}, unit[3] = {0, 0, 0}, item[2] = {0, 0}, ntmax = 16;
    int32_t ntp[2] = {0, 0};
    for (int e = 0; e < E + S; ++e) {
      const int64_t rows = s_cnt[e];
      if (rows == 0) continue;
      const int g = ng++;
      s_gexp[g] = e;
      s_off[g] = (int32_t)off;
      const int nt = pf_ntok_dev(rows);
      ntmax = max(ntmax, nt);
      const int64_t tiles = (rows + nt - 1) / nt;
      // images: phase 1 over d, phase 2 over this expert's f (regions sized with f_max)
      s_o[0][g] = oimg[0];
      oimg[0] += (tiles * (a.d / kPfK) * nt * 128 + 255) & ~int64_t(255);
      s_o[1][g] = oimg[1];
      oimg[1] += (tiles * (a.f_max / kPfK) * nt * 128 + 255) & ~int64_t(255);
      s_blk[0][g] = blk[0];
      blk[0] += (int32_t)(tiles * (a.d / kPfK));
      s_blk[1][g] = blk[1];
      blk[1] += (int32_t)(tiles * (s_shape[e][2][0] / kPfK));
      s_tp[0][g] = ntp[0];
      s_tp[1][g] = ntp[1];
      for (int j = 0; j < 3; ++j) {
        const int mk = s_shape[e][j][0], rank = s_shape[e][j][2], rch = s_shape[e][j][3];
        s_o[2 + j][g] = ot[j];
        s_o[5 + j][g] = op[j];
        s_unit[j][g] = 0;
        if (rank <= 0) continue;
        ot[j] += (tiles * rch * 2 * nt * 128 + 255) & ~int64_t(255);
        const int ks = pf_t_splits_dev(rows, mk, rch, a.sms);
        op[j] += ((int64_t)max(mk / kPfK, ks) * rows * rch * 64 * 4 + 255) & ~int64_t(255);
        const int ph = j == 2 ? 1 : 0;
        s_unit[j][g] = unit[ph];  // unit0 of this t problem (phase-wide prefix)
        unit[ph] += (int32_t)((rows + kTRows - 1) / kTRows) * rch * ks;
        ++ntp[ph];
      }
      s_item[0][g] = item[0];
      item[0] += (int32_t)((s_shape[e][0][1] / kPfM) * tiles);
      s_item[1][g] = item[1];
      item[1] += (int32_t)((s_shape[e][2][1] / kPfM) * tiles);
      off += rows;
    }
    s_ng = ng;
    s_item[0][ng] = item[0];
    s_item[1][ng] = item[1];
    for (int ph = 0; ph < 2; ++ph) {
      int32_t* c = a.counts + 16 * ph;
      c[0] = ng;
      c[1] = blk[ph];
      c[2] = ntp[ph];
      c[3] = unit[ph];
      c[4] = ng;
      c[5] = item[ph];
      c[6] = ntmax;
    }
  }
  __syncthreads();
  const int ng = s_ng;
  // 3. grouped rows: token (x row) and Y slot, entries of an expert in (t, k) order
  for (int g = warp; g < ng; g += nwarps) {
    const int e = s_gexp[g];
    int32_t* tok = a.tok + s_off[g];
    int32_t* slot = a.slot + s_off[g];
    if (e < E) {
      int64_t pos = 0;
      for (int64_t base = 0; base < mK; base += 32) {
        const int64_t i = base + lane;
        const bool hit = i < mK && a.ids[i] == e;
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int64_t p = pos + __popc(b & ((1u << lane) - 1u));
          tok[p] = (int32_t)(i / K);
          slot[p] = (int32_t)i;
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
}

}  // namespace milo_dev
