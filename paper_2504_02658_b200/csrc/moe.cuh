// MoE layer kernels (new: the reference has no MoE layer).
//
//   router_topk_kernel : top-k by descending fp32 logit (ties -> lower id),
//                        softmax weights (Mixtral top-k renorm / DeepSeek all).
//   moe_route_kernel   : one CTA; deterministic counting sort of the (token, k)
//                        entries by expert (ascending token order inside an
//                        expert, warp ballots + fixed-order warp scans), then
//                        the two grouped-GEMM problem tables:
//                          phase 1: per (expert, 16-token block) SwiGLU problem
//                                   over w1|w3 -> h act tiles
//                          phase 2: per block, w2 -> rows of the slot buffer Y
//                        plus zeroed fix-up counters.
//   moe_gather_kernel  : x rows of every block -> binary16 act tiles.
//   moe_combine_kernel : out[t] = sum_k w[t,k] Y[t*K+k] (k order) + shared rows.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "gemv.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace milo_dev {

// ---------------------------------------------------------------------------
// router
// ---------------------------------------------------------------------------
// Top-k of one token's logits by one warp (descending, ties -> lower id) and
// its routing weights (score_mode 0: softmax over the top-k, Mixtral; 1:
// softmax over all experts, DeepSeek).  E <= 256: 8 logits per lane.
__device__ __forceinline__ void topk_regs(const float* __restrict__ l, int E, int K, int score_mode,
                                          int32_t* ids, float* wts, int lane) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < E ? __ldg(l + e) : -INFINITY;
  }
  float mx_all = -INFINITY;
#pragma unroll
  for (int i = 0; i < 8; ++i) mx_all = fmaxf(mx_all, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx_all = fmaxf(mx_all, __shfl_xor_sync(0xffffffffu, mx_all, o));
  uint32_t used = 0u;  // bit i: v[i] of this lane taken
  // the selected (value, id) of step k stay on lane k (K <= 16 < 32): no local arrays
  float my_v = -INFINITY;
  int my_e = -1;
  for (int k = 0; k < K; ++k) {
    float best = -INFINITY;
    int bid = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane + 32 * i;
      if (e < E && !(used >> i & 1u) && (bid == 0x7fffffff || v[i] > best)) {
        best = v[i];
        bid = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oid = __shfl_xor_sync(0xffffffffu, bid, o);
      if (oid != 0x7fffffff && (bid == 0x7fffffff || ov > best || (ov == best && oid < bid))) {
        best = ov;
        bid = oid;
      }
    }
    if ((bid & 31) == lane) used |= 1u << (bid >> 5);
    if (lane == k) {
      my_v = best;
      my_e = bid;
    }
  }
  // weights: lane k < K owns selection k (Mixtral: softmax over the top-k;
  // DeepSeek: softmax over all experts)
  const float top0 = __shfl_sync(0xffffffffu, my_v, 0);
  float num, denom;
  if (score_mode == 0) {
    num = lane < K ? expf(my_v - top0) : 0.0f;
    denom = num;
  } else {
    num = lane < K ? expf(my_v - mx_all) : 0.0f;
    denom = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (lane + 32 * i < E) denom += expf(v[i] - mx_all);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, o);
  if (lane < K) {
    ids[lane] = my_e;
    wts[lane] = num / denom;
  }
}

// One warp per token (the prefill router): topk_regs into ids / wts[t K ...].
__device__ __forceinline__ void topk_warp(const float* __restrict__ l, int64_t t, int E, int K,
                                          int score_mode, int32_t* __restrict__ ids,
                                          float* __restrict__ wts, int lane) {
  topk_regs(l, E, K, score_mode, ids + t * K, wts + t * K, lane);
}

__global__ void router_topk_kernel(const float* __restrict__ logits, int64_t m, int E, int K,
                                   int score_mode, int32_t* __restrict__ ids,
                                   float* __restrict__ wts) {
  pdl_wait();  // logits may come from the preceding grid
  const int warps = blockDim.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
  if (t >= m) return;
  topk_warp(logits + t * E, t, E, K, score_mode, ids, wts, threadIdx.x & 31);
}

// Router GEMM (the MoE gate, x W_gate): logits[t][e] = sum_k half(x[t][k]) *
// gate[e][k] in fp32.  Bit-exact order, restated in oracle/milo_oracle.c
// (or_router_gemm): lane l of the warp owning (t, e) sums the products of
// k = l, l + 32, ... in ascending k (each product of two binary16 values is
// exact in fp32), then the 32 lane sums meet in the xor tree 16, 8, 4, 2, 1.
// The gate rows (E x d binary16) are read once per token block from L2.
__global__ void router_gemm_kernel(const void* __restrict__ x, int32_t x_dtype, int64_t ldx, int64_t m,
                                   int64_t d, const __half* __restrict__ gate, int32_t E,
                                   float* __restrict__ logits) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);  // output index t * E + e
  if (o >= m * E) return;
  const int64_t t = o / E;
  const int e = (int)(o - t * E);
  const __half* g = gate + (int64_t)e * d;
  float acc = 0.0f;
  if (x_dtype == 0) {
    const float* xr = static_cast<const float*>(x) + t * ldx;
    for (int64_t k = lane; k < d; k += 32)
      acc = __fmaf_rn(__half2float(__float2half_rn(xr[k])), __half2float(g[k]), acc);
  } else {
    const __half* xr = static_cast<const __half*>(x) + t * ldx;
    for (int64_t k = lane; k < d; k += 32) acc = __fmaf_rn(__half2float(xr[k]), __half2float(g[k]), acc);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) logits[o] = acc;
}

// ---------------------------------------------------------------------------
// routing -> problem tables
// ---------------------------------------------------------------------------
struct ExpertDev {
  const uint8_t* w[3];       // w1, w3, w2 tiles
  const uint8_t* ucodes[3];
  const float* uscales[3];
  const float* ureal[3];
  const uint8_t* vcodes[3];
  const float* vscales[3];
  const float* vreal[3];
  int32_t rank[3];
  int32_t gpr[3];
  int32_t f;                 // intermediate width of this expert
  int32_t mode;
};

struct MoeRouteArgs {
  const int32_t* ids;        // m x K (-1 = unused)
  int64_t m;
  int32_t K, E, n_shared;
  int32_t d;
  int32_t m_pad;
  const ExpertDev* experts;  // E routed then n_shared shared
  int32_t max_blocks;
  // outputs / workspace
  int32_t* elist;            // entries grouped by expert: entry index (t*K+k) or shared slot
  int32_t* block_expert;     // per block: expert
  int32_t* block_start;      // per block: first position in elist
  GemvProblem* p1;
  GemvProblem* p2;
  int32_t* n_p1;
  int32_t* n_p2;
  uint8_t* act_pool;         // per block: (d/32) * m_pad * 64 bytes
  uint8_t* h_pool;           // per block: (f_max/32) * m_pad * 64 bytes
  int64_t h_block_bytes;
  float* t1_pool;            // per block: 2 x m_pad x rank1_max
  float* t2_pool;            // per block: m_pad x rank2_max
  int32_t rank1_max, rank2_max;
  float* Y;                  // (m*K + n_shared*m) x d fp32
  int32_t* zero_ptr;         // counters to clear
  int64_t zero_count;
  int32_t* n_blocks_out;
  // fused router (optional): logits m x E -> ids / wts (then a.ids == ids_out)
  const float* logits;
  int32_t* ids_out;
  float* wts_out;
  int32_t score_mode;
};

constexpr int kRouteThreads = 1024;
constexpr int kRouteMaxE = 256;

// Publishes the routing ids into mapped pinned host memory, then (after a
// system-scope fence) the call's epoch into a host flag word: the prefill
// planner spins on the flag instead of a D2H copy plus a stream synchronise.
__global__ void publish_ids_kernel(const int32_t* __restrict__ ids, int64_t n, int32_t* __restrict__ host_ids,
                                   volatile int32_t* host_flag, int32_t epoch) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) host_ids[i] = ids[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *host_flag = epoch;
  }
}

__global__ void __launch_bounds__(kRouteThreads) moe_route_kernel(MoeRouteArgs a) {
  pdl_wait();
  __shared__ int32_t wtot[32][kRouteMaxE];  // per-warp per-expert counts of the round
  __shared__ int32_t cnt[kRouteMaxE + 8];
  __shared__ int32_t base[kRouteMaxE + 8];
  __shared__ int32_t off[kRouteMaxE + 8];
  __shared__ int32_t boff[kRouteMaxE + 8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int E = a.E, K = a.K;
  const int ET = E + a.n_shared;
  if (a.logits != nullptr) {  // router: one warp per token
    for (int64_t t = warp; t < a.m; t += blockDim.x >> 5)
      topk_warp(a.logits + t * E, t, E, K, a.score_mode, a.ids_out, a.wts_out, lane);
    __syncthreads();  // ids_out is read back below (block-visible after the barrier)
  }
  for (int64_t i = tid; i < a.zero_count; i += blockDim.x) a.zero_ptr[i] = 0;
  for (int e = tid; e < ET; e += blockDim.x) {
    cnt[e] = e < E ? 0 : (int32_t)a.m;
    base[e] = 0;
  }
  __syncthreads();
  const uint32_t ltmask = (1u << lane) - 1u;
  // pass 0: counts; pass 1: positions (ascending token order within an expert)
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      if (tid == 0) {
        int32_t acc = 0, bacc = 0;
        for (int e = 0; e < ET; ++e) {
          off[e] = acc;
          boff[e] = bacc;
          acc += cnt[e];
          bacc += (cnt[e] + a.m_pad - 1) / a.m_pad;
        }
        off[ET] = acc;
        boff[ET] = bacc;
        *a.n_blocks_out = bacc;
      }
      __syncthreads();
    }
    for (int64_t r0 = 0; r0 < a.m; r0 += blockDim.x) {
      const int64_t t = r0 + tid;
      int32_t my[16];
      for (int k = 0; k < K; ++k) my[k] = (t < a.m) ? a.ids[t * K + k] : -1;
      for (int e = 0; e < E; ++e) {
        int kk = -1;
        for (int k = 0; k < K; ++k)
          if (my[k] == e) kk = k;
        const uint32_t vote = __ballot_sync(0xffffffffu, kk >= 0);
        if (lane == 0) wtot[warp][e] = __popc(vote);
        if (pass == 1 && kk >= 0) my[kk] = -2 - __popc(vote & ltmask);  // stash lane rank
      }
      __syncthreads();
      if (pass == 0) {
        for (int e = tid; e < E; e += blockDim.x) {
          int32_t s = 0;
          for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wtot[w][e];
          cnt[e] += s;
        }
      } else {
        // positions: off[e] + base[e] + (warps before) + lane rank
        for (int k = 0; k < K; ++k) {
          if (t < a.m && my[k] <= -2) {
            const int32_t e = a.ids[t * K + k];
            int32_t before = 0;
            for (int w = 0; w < warp; ++w) before += wtot[w][e];
            const int32_t pos = off[e] + base[e] + before + (-2 - my[k]);
            a.elist[pos] = (int32_t)(t * K + k);
          }
        }
        __syncthreads();
        for (int e = tid; e < E; e += blockDim.x) {
          int32_t s = 0;
          for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wtot[w][e];
          base[e] += s;
        }
      }
      __syncthreads();
    }
  }
  // shared experts: every token, slot m*K + s*m + t
  for (int s = 0; s < a.n_shared; ++s)
    for (int64_t t = tid; t < a.m; t += blockDim.x)
      a.elist[off[E + s] + t] = (int32_t)(a.m * K + s * a.m + t);
  __syncthreads();
  // problem tables: one thread per expert, blocks in order
  for (int e = tid; e < ET; e += blockDim.x) {
    const ExpertDev& ex = a.experts[e];
    const int nb = (cnt[e] + a.m_pad - 1) / a.m_pad;
    for (int b = 0; b < nb; ++b) {
      const int blk = boff[e] + b;
      if (blk >= a.max_blocks) break;
      a.block_expert[blk] = e;
      a.block_start[blk] = off[e] + b * a.m_pad;
      const int rows = min(a.m_pad, cnt[e] - b * a.m_pad);
      GemvProblem p{};
      p.w[0] = ex.w[0];
      p.w[1] = ex.w[1];
      p.act = a.act_pool + (int64_t)blk * (a.d / 32) * a.m_pad * 64;
      for (int mat = 0; mat < 2; ++mat) {
        p.rank[mat] = ex.rank[mat];
        p.vgpr[mat] = ex.gpr[mat];
        p.vcodes[mat] = ex.vcodes[mat];
        p.vscales[mat] = ex.vscales[mat];
        p.vreal[mat] = ex.vreal[mat];
        p.ucodes[mat] = ex.ucodes[mat];
        p.uscales[mat] = ex.uscales[mat];
        p.ureal[mat] = ex.ureal[mat];
        p.t[mat] = ex.rank[mat] > 0
                       ? a.t1_pool + ((int64_t)blk * 2 + mat) * a.m_pad * a.rank1_max
                       : nullptr;
      }
      p.k = a.d;
      p.n = ex.f;
      p.m = rows;
      p.mode = ex.mode;
      p.kind = kSwigluAct;
      p.out = a.h_pool + (int64_t)blk * a.h_block_bytes;
      a.p1[blk] = p;
      GemvProblem q{};
      q.w[0] = ex.w[2];
      q.act = a.h_pool + (int64_t)blk * a.h_block_bytes;
      q.rank[0] = ex.rank[2];
      q.vgpr[0] = ex.gpr[2];
      q.vcodes[0] = ex.vcodes[2];
      q.vscales[0] = ex.vscales[2];
      q.vreal[0] = ex.vreal[2];
      q.ucodes[0] = ex.ucodes[2];
      q.uscales[0] = ex.uscales[2];
      q.ureal[0] = ex.ureal[2];
      q.t[0] = ex.rank[2] > 0 ? a.t2_pool + (int64_t)blk * a.m_pad * a.rank2_max : nullptr;
      q.k = ex.f;
      q.n = a.d;
      q.m = rows;
      q.mode = ex.mode;
      q.kind = kStoreRows;
      q.out_dtype = 0;
      q.ldo = a.d;
      q.out = a.Y;
      q.row_map = a.elist + off[e] + b * a.m_pad;
      a.p2[blk] = q;
    }
  }
  if (tid == 0) {
    const int nb = min(boff[ET], a.max_blocks);
    *a.n_p1 = nb;
    *a.n_p2 = nb;
  }
  pdl_launch_dependents();
}

// x rows of each block -> binary16 act tiles (m_pad rows, zero padded).
__global__ void moe_gather_kernel(const void* __restrict__ x, int32_t x_dtype, int64_t d, int K,
                                  int64_t m, const int32_t* __restrict__ elist,
                                  const int32_t* __restrict__ block_start,
                                  const int32_t* __restrict__ block_expert,
                                  const int32_t* __restrict__ n_blocks, int32_t n_routed,
                                  int32_t m_pad, uint8_t* act_pool, const GemvProblem* __restrict__ p1) {
  // grid (block, row): one row of one block per CTA, 16-byte chunks (8 binary16)
  pdl_wait();
  const int blk = blockIdx.x, r = blockIdx.y;
  if (blk >= *n_blocks) return;
  const int rows = p1[blk].m;
  int32_t tok = -1;
  if (r < rows) {
    const int32_t entry = elist[block_start[blk] + r];
    tok = block_expert[blk] >= n_routed ? (int32_t)((entry - m * K) % m) : entry / K;
  }
  uint4* act = reinterpret_cast<uint4*>(act_pool + (int64_t)blk * (d / 32) * m_pad * 64);
  const int chunks = (int)(d / 8);  // 4 per 32-wide k tile
  const int sw = (r >> 1) & 3;      // act-tile swizzle moves whole 16-byte chunks
  for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (tok >= 0) {
      if (x_dtype == 0) {
        const float4* src = reinterpret_cast<const float4*>(x) + ((int64_t)tok * d) / 4 + 2 * c;
        const float4 a = src[0], b = src[1];
        v.x = h2_as_u32(__floats2half2_rn(a.x, a.y));
        v.y = h2_as_u32(__floats2half2_rn(a.z, a.w));
        v.z = h2_as_u32(__floats2half2_rn(b.x, b.y));
        v.w = h2_as_u32(__floats2half2_rn(b.z, b.w));
      } else {
        v = reinterpret_cast<const uint4*>(x)[((int64_t)tok * d) / 8 + c];
      }
    }
    const int kt = c >> 2, ch = c & 3;
    act[(int64_t)kt * (m_pad * 4) + r * 4 + (ch ^ sw)] = v;
  }
  pdl_launch_dependents();
}

__global__ void moe_combine_kernel(const float* __restrict__ Y, const int32_t* __restrict__ ids,
                                   const float* __restrict__ wts, int64_t m, int K, int n_shared,
                                   int64_t d, void* out, int32_t out_dtype) {
  pdl_wait();
  const int64_t total = m * (d / 4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / (d / 4), c4 = i % (d / 4);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < K; ++k) {
      if (ids[t * K + k] < 0) continue;
      const float w = wts[t * K + k];
      const float4 y = reinterpret_cast<const float4*>(Y + (t * K + k) * d)[c4];
      acc.x += w * y.x;
      acc.y += w * y.y;
      acc.z += w * y.z;
      acc.w += w * y.w;
    }
    for (int s = 0; s < n_shared; ++s) {
      const float4 y = reinterpret_cast<const float4*>(Y + (m * K + s * m + t) * d)[c4];
      acc.x += 1.0f * y.x;
      acc.y += 1.0f * y.y;
      acc.z += 1.0f * y.z;
      acc.w += 1.0f * y.w;
    }
    if (out_dtype == 0) {
      reinterpret_cast<float4*>(out)[i] = acc;
    } else {
      __half2* o = reinterpret_cast<__half2*>(out) + i * 2;
      o[0] = __floats2half2_rn(acc.x, acc.y);
      o[1] = __floats2half2_rn(acc.z, acc.w);
    }
  }
}

}  // namespace milo_dev

namespace milo_dev {

// ---------------------------------------------------------------------------
// Expert-parallel fixed-capacity exchange (paper_2504_02658_b200/ep.py):
// entry e = t K + k with expert id >= 0 goes to rank id / per, at position
// pos = #{entries e' < e with the same destination}; row slot dest * C + pos of
// the send buffer carries binary16 x[t] and the local expert id (-1 = unused).
// One CTA (entries <= 1024).  slot[e] = dest * C + pos (or -1) for the combine.
// ---------------------------------------------------------------------------
// ld_send: row stride of send_x (halves).  send_meta == null: the local expert id
// travels in the row itself (int32 at half-column d; ld_send >= d + 8), so one
// all-to-all moves rows and ids together.
__global__ void ep_dispatch_kernel(const int32_t* __restrict__ ids, int32_t mK, int32_t K, int32_t W,
                                   int32_t per, int32_t C, const void* __restrict__ x, int32_t x_dtype,
                                   int64_t d, __half* __restrict__ send_x, int64_t ld_send,
                                   int32_t* __restrict__ send_meta, int32_t* __restrict__ slot) {
  __shared__ int32_t s_slot[1024];
  __shared__ int32_t s_src[1024 * 8];  // slot -> entry (W * C <= 8192)
  const int tid = threadIdx.x;
  for (int i = tid; i < W * C; i += blockDim.x) s_src[i] = -1;
  __syncthreads();
  for (int e = tid; e < mK; e += blockDim.x) {
    const int id = ids[e];
    int sl = -1;
    if (id >= 0) {
      const int dest = id / per;
      int pos = 0;
      for (int e2 = 0; e2 < e; ++e2) {
        const int id2 = ids[e2];
        pos += (id2 >= 0 && id2 / per == dest);
      }
      sl = dest * C + pos;
      s_src[sl] = e;
    }
    s_slot[e] = sl;
    slot[e] = sl;
  }
  __syncthreads();
  for (int r = tid; r < W * C; r += blockDim.x) {
    const int e = s_src[r];
    const int32_t lid = e >= 0 ? ids[e] - (ids[e] / per) * per : -1;
    if (send_meta != nullptr) {
      send_meta[r] = lid;
    } else {
      int32_t* tail = reinterpret_cast<int32_t*>(send_x + (int64_t)r * ld_send + d);
      tail[0] = lid;
      tail[1] = tail[2] = tail[3] = 0;
    }
  }
  const int64_t d8 = d / 8;
  for (int64_t i = tid; i < (int64_t)W * C * d8; i += blockDim.x) {
    const int r = (int)(i / d8), c = (int)(i % d8) * 8;
    const int e = s_src[r];
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (e >= 0) {
      const int64_t t = e / K;
      if (x_dtype == 0) {
        const float4* s = reinterpret_cast<const float4*>(static_cast<const float*>(x) + t * d + c);
        const float4 p0 = s[0], p1 = s[1];
        v = make_uint4(h2_as_u32(__floats2half2_rn(p0.x, p0.y)), h2_as_u32(__floats2half2_rn(p0.z, p0.w)),
                       h2_as_u32(__floats2half2_rn(p1.x, p1.y)), h2_as_u32(__floats2half2_rn(p1.z, p1.w)));
      } else {
        v = *reinterpret_cast<const uint4*>(static_cast<const __half*>(x) + t * d + c);
      }
    }
    *reinterpret_cast<uint4*>(send_x + (int64_t)r * ld_send + c) = v;
  }
  (void)s_slot;
}

// out[t] = sum_k w[t,k] y[slot[t K + k]] (k order, moe_combine semantics), f32.
// extra (nullable): m x d f32 added after the routed sum (the shared experts).
__global__ void ep_combine_kernel(const float* __restrict__ y, const int32_t* __restrict__ slot,
                                  const float* __restrict__ wts, int64_t m, int32_t K, int64_t d,
                                  float* __restrict__ out, const float* __restrict__ extra) {
  const int64_t total = m * (d / 4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / (d / 4), c4 = i % (d / 4);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < K; ++k) {
      const int sl = slot[t * K + k];
      if (sl < 0) continue;
      const float w = wts[t * K + k];
      const float4 v = reinterpret_cast<const float4*>(y + (int64_t)sl * d)[c4];
      acc.x += w * v.x;
      acc.y += w * v.y;
      acc.z += w * v.z;
      acc.w += w * v.w;
    }
    if (extra != nullptr) {
      const float4 v = reinterpret_cast<const float4*>(extra)[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(out)[i] = acc;
  }
}

// Received EP rows (ld halves, the local expert id as int32 at half-column d)
// -> contiguous binary16 rows + ids + unit weights for the local grouped call.
__global__ void ep_unpack_kernel(const __half* __restrict__ recv, int64_t rows, int64_t d, int64_t ld,
                                 __half* __restrict__ x, int32_t* __restrict__ lids, float* __restrict__ ones) {
  const int64_t d8 = d / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * (d8 + 1);
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (d8 + 1), c = i % (d8 + 1);
    if (c < d8) {
      reinterpret_cast<uint4*>(x + r * d)[c] = reinterpret_cast<const uint4*>(recv + r * ld)[c];
    } else {
      lids[r] = *reinterpret_cast<const int32_t*>(recv + r * ld + d);
      ones[r] = 1.0f;
    }
  }
}

}  // namespace milo_dev
