// Expert-parallel MoE layer, C++ host over NCCL.
//
// Rank r of W owns the routed experts [r per, (r + 1) per), per = ceil(E / W);
// shared experts are replicated.  One call on a rank's m local tokens, all
// stream-ordered on the caller's stream (no host synchronisation):
//   1. router top-k of the local logits (router_topk_kernel; bit-exact ids);
//   2. dispatch (ep_dispatch_kernel): every routed entry becomes a binary16 row
//      of a fixed-capacity send buffer, C rows per destination rank, the local
//      expert id riding in the row (int32 at half-column d; -1 = unused row);
//   3. exchange: one grouped ncclSend / ncclRecv per peer (NCCL has no
//      all-to-all, nccl.h ncclSend / ncclRecv);
//   4. the owned experts on the received rows (milo_moe_forward_routed of the
//      rank's local layer, top_k = 1, weight 1): the same decode / prefill
//      kernels as the single-GPU layer;
//   5. the inverse exchange returns every entry's fp32 expert output;
//   6. combine (ep_combine_kernel): sum_k w_k y_k in k order, plus the shared
//      experts' output computed locally (milo_moe_forward of the shared layer).
//
// NCCL is resolved at run time (dlopen / dlsym of libnccl.so.2, reusing the copy
// already loaded into the process, e.g. torch's), so the library has no link-time
// NCCL dependency and the rest of the ABI works without it.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = "libnccl.so.2 not found";
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
             sym(api.CommDestroy, "ncclCommDestroy") && sym(api.CommCount, "ncclCommCount") &&
             sym(api.CommUserRank, "ncclCommUserRank") && sym(api.Send, "ncclSend") && sym(api.Recv, "ncclRecv") &&
             sym(api.GroupStart, "ncclGroupStart") && sym(api.GroupEnd, "ncclGroupEnd") &&
             sym(api.GetErrorString, "ncclGetErrorString");
    if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

#define NCCL_TRY(call)                                                                  \
  do {                                                                                  \
    const ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess) return fail(MILO_ERR_CUDA, "nccl: %s", nccl().GetErrorString(r_)); \
  } while (0)

}  // namespace

struct milo_ep_layer {
  milo_moe* local = nullptr;   // owned routed experts (top_k = 1), may be null (rank owns none)
  milo_moe* shared = nullptr;  // replicated shared experts, may be null
  int32_t E = 0, K = 0, score_mode = 0, world = 1, rank = 0, per = 1, d = 0;
  ncclComm_t comm = nullptr;
};

extern "C" milo_status milo_ep_unique_id(uint8_t* id, int64_t id_bytes) {
  if (!id || id_bytes < (int64_t)sizeof(ncclUniqueId)) return fail(MILO_ERR_ARGUMENT, "need a 128-byte id buffer");
  if (!nccl().ok) return fail(MILO_ERR_CUDA, "%s", nccl().err.c_str());
  ncclUniqueId u;
  NCCL_TRY(nccl().GetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return MILO_OK;
}

extern "C" milo_status milo_ep_comm_create(const uint8_t* id, int32_t world, int32_t rank, void** comm) {
  if (!id || !comm || world < 1 || rank < 0 || rank >= world) return fail(MILO_ERR_ARGUMENT, "bad communicator args");
  if (!nccl().ok) return fail(MILO_ERR_CUDA, "%s", nccl().err.c_str());
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  NCCL_TRY(nccl().CommInitRank(&c, world, u, rank));
  *comm = c;
  return MILO_OK;
}

extern "C" milo_status milo_ep_comm_destroy(void* comm) {
  if (!comm) return MILO_OK;
  if (!nccl().ok) return fail(MILO_ERR_CUDA, "%s", nccl().err.c_str());
  NCCL_TRY(nccl().CommDestroy(static_cast<ncclComm_t>(comm)));
  return MILO_OK;
}

extern "C" milo_status milo_ep_layer_create(milo_moe* local, milo_moe* shared, int32_t n_experts, int32_t top_k,
                                            int32_t score_mode, void* comm, milo_ep_layer** out) {
  if (!out || !comm) return fail(MILO_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (!nccl().ok) return fail(MILO_ERR_CUDA, "%s", nccl().err.c_str());
  if (n_experts < 1 || top_k < 1 || top_k > 16 || top_k > n_experts) return fail(MILO_ERR_CONFIG, "bad E / top_k");
  if (score_mode != 0 && score_mode != 1) return fail(MILO_ERR_CONFIG, "unknown score mode");
  int world = 0, rank = 0;
  NCCL_TRY(nccl().CommCount(static_cast<ncclComm_t>(comm), &world));
  NCCL_TRY(nccl().CommUserRank(static_cast<ncclComm_t>(comm), &rank));
  const int per = (n_experts + world - 1) / world;
  const int owned = std::max(0, std::min(n_experts, (rank + 1) * per) - rank * per);
  if ((local ? local->E : 0) != owned)
    return fail(MILO_ERR_CONFIG, "rank %d of %d owns %d experts, the local layer has %d", rank, world, owned,
                local ? local->E : 0);
  if (local && local->K != 1) return fail(MILO_ERR_CONFIG, "the local layer must be top_k = 1");
  if (shared && shared->E != 0) return fail(MILO_ERR_CONFIG, "the shared layer must hold shared experts only");
  if (!local && !shared) return fail(MILO_ERR_CONFIG, "no experts on this rank");
  auto* L = new milo_ep_layer();
  L->local = local;
  L->shared = shared;
  L->E = n_experts;
  L->K = top_k;
  L->score_mode = score_mode;
  L->world = world;
  L->rank = rank;
  L->per = per;
  L->d = local ? local->d : shared->d;
  L->comm = static_cast<ncclComm_t>(comm);
  if (local && shared && local->d != shared->d) {
    delete L;
    return fail(MILO_ERR_SHAPE, "local / shared hidden sizes differ");
  }
  *out = L;
  return MILO_OK;
}

extern "C" milo_status milo_ep_layer_destroy(milo_ep_layer* L) {
  delete L;
  return MILO_OK;
}

extern "C" milo_status milo_ep_forward(milo_ep_layer* L, const void* x, int64_t m, int32_t x_dtype,
                                       const float* logits, float* out, int32_t capacity, void* stream_) {
  if (!L) return fail(MILO_ERR_ARGUMENT, "null layer");
  if (m < 0) return fail(MILO_ERR_SHAPE, "negative token count");
  if (x_dtype != MILO_F32 && x_dtype != MILO_F16) return fail(MILO_ERR_ARGUMENT, "x dtype");
  if (m > 0 && (!x || !logits || !out)) return fail(MILO_ERR_ARGUMENT, "null argument");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int K = L->K, W = L->world, d = L->d;
  // every rank must issue the same exchange: C = the caller's capacity (the
  // largest m K of the group), or m K when the caller runs equal batches
  const int64_t C = capacity > 0 ? capacity : m * K;
  if (m * K > C) return fail(MILO_ERR_CONFIG, "capacity %lld < m * top_k = %lld", (long long)C, (long long)(m * K));
  if (m * K > 1024 || (int64_t)W * C > 8192) return fail(MILO_ERR_CONFIG, "EP exchange: m K <= 1024, W C <= 8192");
  if (d % 8 != 0) return fail(MILO_ERR_SHAPE, "d must be a multiple of 8");
  const int64_t ld = d + 8, rows = (int64_t)W * C;
  Arena ar;
  const size_t o_ids = ar.take((size_t)std::max<int64_t>(m * K, 1) * 4);
  const size_t o_w = ar.take((size_t)std::max<int64_t>(m * K, 1) * 4);
  const size_t o_slot = ar.take((size_t)std::max<int64_t>(m * K, 1) * 4);
  const size_t o_send = ar.take((size_t)rows * ld * 2);
  const size_t o_recv = ar.take((size_t)rows * ld * 2);
  const size_t o_x = ar.take((size_t)rows * d * 2);
  const size_t o_lid = ar.take((size_t)rows * 4);
  const size_t o_one = ar.take((size_t)rows * 4);
  const size_t o_y = ar.take((size_t)rows * d * 4);
  const size_t o_yb = ar.take((size_t)rows * d * 4);
  const size_t o_sh = ar.take(L->shared ? (size_t)std::max<int64_t>(m, 1) * d * 4 : 0);
  void* mem = nullptr;
  if (rows > 0) CUDA_TRY(cudaMallocAsync(&mem, ar.size, stream));  // per call, stream-ordered
  uint8_t* b = static_cast<uint8_t*>(mem);
  auto* ids = reinterpret_cast<int32_t*>(b + o_ids);
  auto* wts = reinterpret_cast<float*>(b + o_w);
  auto* slot = reinterpret_cast<int32_t*>(b + o_slot);
  auto* send = reinterpret_cast<__half*>(b + o_send);
  auto* recv = reinterpret_cast<__half*>(b + o_recv);
  auto* xr = reinterpret_cast<__half*>(b + o_x);
  auto* lid = reinterpret_cast<int32_t*>(b + o_lid);
  auto* one = reinterpret_cast<float*>(b + o_one);
  auto* y = reinterpret_cast<float*>(b + o_y);
  auto* yb = reinterpret_cast<float*>(b + o_yb);
  auto* sh = reinterpret_cast<float*>(b + o_sh);
  milo_status st = MILO_OK;
  auto guard = [&](cudaError_t e) {
    if (e != cudaSuccess && st == MILO_OK) st = fail(MILO_ERR_CUDA, "ep: %s", cudaGetErrorString(e));
  };
  auto nguard = [&](ncclResult_t r) {
    if (r != ncclSuccess && st == MILO_OK) st = fail(MILO_ERR_CUDA, "nccl: %s", nccl().GetErrorString(r));
  };
  if (m > 0) {
    guard(launch(router_topk_kernel, dim3((unsigned)((m + 7) / 8)), dim3(256), 0, stream, false, logits, m, L->E, K,
                 L->score_mode, ids, wts));
    guard(launch(ep_dispatch_kernel, dim3(1), dim3(1024), 0, stream, false, (const int32_t*)ids, (int32_t)(m * K), K,
                 W, L->per, (int32_t)C, x, x_dtype, (int64_t)d, send, ld, (int32_t*)nullptr, slot));
  } else if (rows > 0) {
    guard(cudaMemsetAsync(send, 0xFF, (size_t)rows * ld * 2, stream));  // every row unused (id -1)
  }
  // exchange 1: C rows of (d + 8) halves to / from every peer
  if (st == MILO_OK && rows > 0) {
    const size_t bytes = (size_t)C * ld * 2;
    nguard(nccl().GroupStart());
    for (int p = 0; p < W; ++p) {
      nguard(nccl().Send(send + (size_t)p * C * ld, bytes, ncclUint8, p, L->comm, stream));
      nguard(nccl().Recv(recv + (size_t)p * C * ld, bytes, ncclUint8, p, L->comm, stream));
    }
    nguard(nccl().GroupEnd());
  }
  // owned experts on the received rows (unused rows carry id -1 and are skipped)
  if (st == MILO_OK && rows > 0) {
    if (L->local) {
      const int64_t n8 = rows * (d / 8 + 1);
      guard(launch(ep_unpack_kernel, dim3((unsigned)std::min<int64_t>((n8 + 255) / 256, 1184)), dim3(256), 0, stream,
                   false, (const __half*)recv, rows, (int64_t)d, ld, xr, lid, one));
      if (st == MILO_OK) st = milo_moe_forward_routed(L->local, xr, rows, MILO_F16, lid, one, y, MILO_F32, stream);
    } else {
      guard(cudaMemsetAsync(y, 0, (size_t)rows * d * 4, stream));
    }
  }
  // exchange 2: the fp32 expert outputs back to their tokens' ranks
  if (st == MILO_OK && rows > 0) {
    const size_t bytes = (size_t)C * d * 4;
    nguard(nccl().GroupStart());
    for (int p = 0; p < W; ++p) {
      nguard(nccl().Send(y + (size_t)p * C * d, bytes, ncclUint8, p, L->comm, stream));
      nguard(nccl().Recv(yb + (size_t)p * C * d, bytes, ncclUint8, p, L->comm, stream));
    }
    nguard(nccl().GroupEnd());
  }
  if (st == MILO_OK && m > 0) {
    if (L->shared) st = milo_moe_forward(L->shared, x, m, x_dtype, nullptr, sh, MILO_F32, nullptr, nullptr, stream);
    const int64_t total = m * (d / 4);
    if (st == MILO_OK)
      guard(launch(ep_combine_kernel, dim3((unsigned)std::min<int64_t>((total + 255) / 256, 1184)), dim3(256), 0,
                   stream, false, (const float*)yb, (const int32_t*)slot, (const float*)wts, m, K, (int64_t)d, out,
                   L->shared ? (const float*)sh : (const float*)nullptr));
  }
  if (mem) guard(cudaFreeAsync(mem, stream));
  return st;
}
