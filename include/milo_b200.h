/*
 * milo_b200.h — C ABI of the B200 (sm_100a) MiLo INT3 + LoRC hot path.
 *
 * Drop-in boundary for the reference's operator
 *
 *   WeightMatrix milo::gemm_w3a16(const WeightMatrix& A, const PackedInt3Matrix& Wp,
 *                                 const std::optional<Compensator>& comp,
 *                                 const GemmConfig& cfg);
 *   (/root/reference/proj/include/milo/gemm.hpp:43-48, src/gemm.cpp:117-199)
 *
 * plus the top-k routed grouped-expert call the reference lacks (SURVEY.md
 * section 8b).  Plain pointers and sizes only; no C++ or torch types.  The
 * C++ host API in milo_b200.hpp mirrors the reference's types on top of this.
 *
 * Conventions
 *  - Device pointers unless a function name ends in _host.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *    device-pointer calls are stream-ordered and never synchronize the host.
 *  - Handles are immutable after creation and may be shared across streams and
 *    threads.
 *  - Workspace: the library keeps one scratch region per (device, stream) it is
 *    called on (allocated stream-ordered with cudaMallocAsync, grown on demand,
 *    reused by later calls on that stream; fresh regions are initialised on the
 *    stream before first use).  milo_stream_release(stream) frees them, e.g.
 *    before the caller destroys the stream.
 *  - Errors: every function returns milo_status; milo_last_error() returns a
 *    thread-local message for the last failure on the calling thread.  Input
 *    validation follows the reference's order (gemm.cpp:120-139) so the same
 *    bad input yields the same category (errors.hpp:9-20).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns MILO_ERR_CUDA.
 */
#ifndef MILO_B200_H
#define MILO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MILO_B200_ABI_VERSION 2

/* milo::ErrorCode (errors.hpp:9-20) in order, offset by one; plus CUDA. */
typedef enum milo_status {
  MILO_OK = 0,
  MILO_ERR_FORMAT = 1,
  MILO_ERR_DATA = 2,
  MILO_ERR_IO = 3,
  MILO_ERR_SHAPE = 4,
  MILO_ERR_RANK = 5,
  MILO_ERR_NUMERIC = 6,
  MILO_ERR_STAT = 7,
  MILO_ERR_PLAN = 8,
  MILO_ERR_RANGE = 9,
  MILO_ERR_CONFIG = 10,
  MILO_ERR_CUDA = 100,
  MILO_ERR_ARGUMENT = 101
} milo_status;

typedef enum milo_layout { MILO_LAYOUT_LINEAR = 0, MILO_LAYOUT_TILED16X64 = 1 } milo_layout;
typedef enum milo_mode { MILO_MODE_SYMMETRIC = 0, MILO_MODE_ASYMMETRIC = 1 } milo_mode;
typedef enum milo_dtype { MILO_F32 = 0, MILO_F16 = 1 } milo_dtype;
typedef enum milo_comp_storage { MILO_COMP_REAL = 0, MILO_COMP_SYMM_INT3 = 1 } milo_comp_storage;
typedef enum milo_score_mode {
  MILO_SCORE_SOFTMAX_TOPK = 0, /* Mixtral: softmax over the selected top-k logits */
  MILO_SCORE_SOFTMAX_ALL = 1   /* DeepSeek: softmax over all experts, no renorm  */
} milo_score_mode;

typedef struct milo_weight milo_weight;
typedef struct milo_comp milo_comp;
typedef struct milo_moe milo_moe;

/* Host-side view of milo::PackedInt3Matrix (pack.hpp:45-66), fields verbatim.
 * rows = k (reduction), cols = n (output).  words holds 3 u32 per 32-code
 * group when !split; plane_a (2 per group) + plane_b (1 per group) when split.
 * scales/zeros are binary16 bit patterns, one per group_size consecutive
 * elements of a row; zeros == NULL means "empty" (symmetric weights).
 * The n_* lengths are element counts of the corresponding arrays. */
typedef struct milo_packed_desc {
  uint64_t rows, cols;
  int32_t layout;     /* milo_layout */
  int32_t split;      /* bool */
  int32_t mode;       /* milo_mode */
  uint64_t group_size;
  const uint32_t* words;
  uint64_t n_words;
  const uint32_t* plane_a;
  uint64_t n_plane_a;
  const uint32_t* plane_b;
  uint64_t n_plane_b;
  const uint16_t* scales;
  uint64_t n_scales;
  const uint16_t* zeros;
  uint64_t n_zeros;
} milo_packed_desc;

/* Host-side view of milo::Compensator (lowrank.hpp:31-50): U is rows x rank,
 * V is rank x cols (real storage), or symm-int3 codes qU (rows x rank) and
 * qVt = V^T (cols x rank) with float scales per group along rank. */
typedef struct milo_comp_desc {
  uint64_t rows, cols, rank;
  int32_t storage; /* milo_comp_storage */
  const float* U;
  const float* V;
  const uint8_t* qu_codes;
  const float* qu_scales;
  const uint8_t* qvt_codes;
  const float* qvt_scales;
  uint64_t group_size; /* symm-int3 grouping along rank */
} milo_comp_desc;

/* milo::GemmConfig (gemm.hpp:17-25).  tile_k/tile_n/pipeline_depth are
 * validated exactly like the reference (gemm.cpp:23-30,131-134); the sm_100a
 * kernels choose their own tiling. */
typedef struct milo_gemm_config {
  int32_t tile_k, tile_n;
  uint64_t group_size;
  int32_t mode;
  int32_t pipeline_depth;
  int32_t materialize_compensator;
} milo_gemm_config;

/* ---------------------------------------------------------------- errors */
const char* milo_last_error(void);
const char* milo_status_name(milo_status s);
int milo_abi_version(void);
/* Probes the current device; MILO_OK iff it is sm_100 and the kernels load. */
milo_status milo_device_check(void);

/* ----------------------------------------------------- weights (pack.hpp) */
/* Validates desc, uploads it and repacks it on the device into the kernel
 * layout (fragment-native 64(n) x 32(k) macro tiles, 896 B each = 0.4375 B
 * per weight).  Blocking. */
milo_status milo_weight_create(const milo_packed_desc* desc, milo_weight** out);
milo_status milo_weight_destroy(milo_weight* w);
milo_status milo_weight_info(const milo_weight* w, uint64_t* rows, uint64_t* cols,
                             int32_t* mode, uint64_t* device_bytes);
/* Device unpack to logical row-major codes (== milo::unpack_codes,
 * pack.cpp:196-211), out: rows*cols bytes. */
milo_status milo_unpack_codes(const milo_weight* w, uint8_t* out, void* stream);
/* Device de-quantization to logical binary16 (== milo::dequant_packed_half,
 * pack.cpp:244-295, bit-exact), out: rows*cols u16.  `mode` must equal the
 * weight's mode (the reference would throw ConfigError on a missing zero). */
milo_status milo_dequant_half(const milo_weight* w, int32_t mode, uint16_t* out, void* stream);

/* ---------------------------------------------- compensator (lowrank.hpp) */
milo_status milo_comp_create(const milo_comp_desc* desc, milo_comp** out);
milo_status milo_comp_destroy(milo_comp* c);
/* The Compensator's rows (k), cols (n), rank and storage (lowrank.hpp:31-50). */
milo_status milo_comp_info(const milo_comp* c, uint64_t* rows, uint64_t* cols, uint64_t* rank,
                           int32_t* storage);

/* --------------------------------------------------- the W3A16 GEMM (K2) */
/* C[m x n] = A_f16[m x k] * (dequant(W) + U V), fp32 accumulation.
 * A: m x a_cols row-major (a_dtype; f32 inputs are rounded to binary16 on the
 * device exactly like gemm.cpp:144-146).  C: m x n row-major (c_dtype).
 * comp may be NULL (== std::nullopt).  m == 0 is a no-op. */
milo_status milo_gemm_w3a16(const milo_weight* w, const milo_comp* comp,
                            const milo_gemm_config* cfg, const void* A, int64_t m,
                            int64_t a_cols, int32_t a_dtype, void* C, int32_t c_dtype,
                            void* stream);
/* Same with host fp32 buffers (the reference's by-value semantics); copies in,
 * runs, copies out, synchronizes.  The end-to-end entry point. */
milo_status milo_gemm_w3a16_host(const milo_weight* w, const milo_comp* comp,
                                 const milo_gemm_config* cfg, const float* A, int64_t m,
                                 int64_t a_cols, float* C);

/* ------------------------------------------- top-k routed MoE layer (new) */
/* One expert = w1 (d x f), w3 (d x f), w2 (f x d) in the reference's k x n
 * orientation (synth.cpp:37-39), each with an optional compensator of its own
 * rank (ragged ranks allowed, 0 == none). */
typedef struct milo_expert_desc {
  const milo_weight* w1;
  const milo_weight* w3;
  const milo_weight* w2;
  const milo_comp* c1;
  const milo_comp* c3;
  const milo_comp* c2;
} milo_expert_desc;

/* Shared experts run on every token with weight 1 (DeepSeek-MoE). */
milo_status milo_moe_create(const milo_expert_desc* experts, int32_t n_experts,
                            const milo_expert_desc* shared, int32_t n_shared, int32_t top_k,
                            int32_t score_mode, milo_moe** out);
milo_status milo_moe_destroy(milo_moe* moe);

/* Router: top-k by descending fp32 logit (ties -> lower expert id), weights
 * per score_mode.  logits m x E; ids/weights m x K. */
milo_status milo_router_topk(const float* logits, int64_t m, int32_t n_experts, int32_t top_k,
                             int32_t score_mode, int32_t* topk_ids, float* topk_w, void* stream);

/* out[m x d] = sum_k w_k * FFN_{e_k}(x) + sum_s FFN_s(x), FFN(x) =
 * (silu(x W1 + x U1 V1) * (x W3 + x U3 V3)) W2 + (h U2) V2.
 * x: m x d (x_dtype), router_logits: m x E fp32.  topk_ids/topk_w are
 * optional outputs (may be NULL). */
milo_status milo_moe_forward(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype,
                             const float* router_logits, void* out, int32_t out_dtype,
                             int32_t* topk_ids, float* topk_w, void* stream);
/* Same with routing given (ids m x K int32, -1 = unused slot; weights m x K). */
milo_status milo_moe_forward_routed(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype,
                                    const int32_t* topk_ids, const float* topk_w, void* out,
                                    int32_t out_dtype, void* stream);
/* The MoE gate (router GEMM, x W_gate): logits[t][e] = sum_k half(x[t][k]) *
 * gate[e][k] in fp32, in a fixed order restated bit-exactly by the oracle
 * (oracle/milo_oracle.c or_router_gemm).  x: m x d (x_dtype) device rows,
 * gate: E x d binary16 (device), logits: m x E fp32 (device). */
milo_status milo_router_gemm(const void* x, int64_t m, int64_t d, int32_t x_dtype, const uint16_t* gate,
                             int32_t n_experts, float* logits, void* stream);
/* Attaches the gate weights (E x d binary16 bits, host memory; uploaded,
 * blocking) to a layer so that milo_moe_forward_x routes from x itself.
 * MILO_ERR_SHAPE unless E and d are the layer's. */
milo_status milo_moe_set_gate(milo_moe* moe, const uint16_t* gate, int64_t n_experts, int64_t d);
/* The whole MoE block from x: router GEMM -> top-k -> experts -> combine.
 * MILO_ERR_CONFIG if no gate was attached.  topk_ids / topk_w optional. */
milo_status milo_moe_forward_x(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype, void* out,
                               int32_t out_dtype, int32_t* topk_ids, float* topk_w, void* stream);

/* Host-buffer end-to-end call: x (m x x_cols f32) and logits (m x logit_cols
 * f32) in host memory, out (m x d f32) host; blocking.  MILO_ERR_SHAPE unless
 * x_cols == d and logit_cols == E (checked before any buffer is touched). */
milo_status milo_moe_forward_host(milo_moe* moe, const float* x, int64_t m, int64_t x_cols,
                                  const float* router_logits, int64_t logit_cols, float* out);

/* ---------------------------------------------- MILO1 container loaders
 * The reference's tensor-store container (tensor_store.cpp:96-131): "MILO1",
 * u32 LE header length, JSON header, little-endian payload.
 * milo_packed_load_host: a packed-i3 container (pack.cpp:306-400, validated
 * like milo::load_packed) into a host desc; the returned handle owns the
 * arrays the desc points to (milo_packed_host_free).  No device needed.
 * milo_weight_load: the same, uploaded and repacked (milo_weight_create).
 * milo_comp_load: the compensator factor pair the reference's quantize writes
 * (<name>.u.milo / <name>.v.milo, pipeline.cpp:233-283; the reference has no
 * reader): symm-i3 codes + binary16 scales (the writer's rounding of the
 * float scales is kept), or f32 real factors.  Errors: MILO_ERR_IO (open),
 * MILO_ERR_FORMAT (magic, header, dtype, payload size), MILO_ERR_SHAPE. */
milo_status milo_packed_load_host(const char* path, milo_packed_desc* desc, void** handle);
void milo_packed_host_free(void* handle);
milo_status milo_weight_load(const char* path, milo_weight** out);
milo_status milo_comp_load(const char* u_path, const char* v_path, milo_comp** out);

/* Expert-parallel exchange (paper_2504_02658_b200/ep.py): fixed-capacity
 * dispatch of the m x K routed entries to `world` ranks owning `per` experts
 * each.  send_x: (world * capacity) rows of ld_send binary16 (the first d =
 * x row), send_meta: local expert id per row (-1 = unused) -- or NULL to put
 * the id in the row itself as an int32 at half-column d (ld_send >= d + 8, one
 * all-to-all for rows and ids); slot: m * K row index of each entry (-1 =
 * unused).  m * K <= 1024, world * capacity <= 8192. */
milo_status milo_ep_dispatch(const int32_t* ids, int64_t m, int32_t K, int32_t world, int32_t per,
                             int32_t capacity, const void* x, int32_t x_dtype, int64_t d, void* send_x,
                             int64_t ld_send, int32_t* send_meta, int32_t* slot, void* stream);
/* out[t] = sum_k w[t,k] y[slot[t K + k]] in k order (f32), the EP combine. */
milo_status milo_ep_combine(const float* y, const int32_t* slot, const float* wts, int64_t m, int32_t K,
                            int64_t d, float* out, void* stream);

/* Frees the scratch regions kept for (current device, stream) after the
 * stream's pending work (synchronizes that stream).  A later call on the same
 * stream allocates them again. */
milo_status milo_stream_release(void* stream);

/* ------------------------------------- expert-parallel layer (NCCL, new)
 * Rank r of W owns routed experts [r*per, (r+1)*per), per = ceil(E / W);
 * shared experts are replicated.  NCCL is resolved at run time (libnccl.so.2
 * already loaded into the process, else dlopen); without it these return
 * MILO_ERR_CUDA.  comm is an ncclComm_t (the caller's, or milo_ep_comm_create
 * from an id made by milo_ep_unique_id on one rank and broadcast). */
typedef struct milo_ep_layer milo_ep_layer;
milo_status milo_ep_unique_id(uint8_t* id, int64_t id_bytes); /* id_bytes >= 128 */
milo_status milo_ep_comm_create(const uint8_t* id, int32_t world, int32_t rank, void** comm);
milo_status milo_ep_comm_destroy(void* comm);
/* local: a layer over this rank's owned experts with top_k = 1 (NULL if it owns
 * none); shared: a layer holding only the shared experts (NULL if none). */
milo_status milo_ep_layer_create(milo_moe* local, milo_moe* shared, int32_t n_experts, int32_t top_k,
                                 int32_t score_mode, void* comm, milo_ep_layer** out);
milo_status milo_ep_layer_destroy(milo_ep_layer* layer);
/* One layer call on this rank's m tokens (x m x d, logits m x E fp32, out m x d
 * fp32, device).  Fixed-capacity exchange: capacity rows per peer, >= m * top_k
 * on every rank and equal across ranks (<= 0: m * top_k, equal batches).
 * Stream-ordered; every rank of the communicator must call it. */
milo_status milo_ep_forward(milo_ep_layer* layer, const void* x, int64_t m, int32_t x_dtype, const float* logits,
                            float* out, int32_t capacity, void* stream);

/* Kernel launches recorded by this library on the calling thread (for the
 * bench's gpu_launches claim). */
uint64_t milo_launch_count(void);

/* Optional CUDA-event timing of the library's own kernels on the launching
 * stream (calling thread only).  kind: 0 grouped GEMM phase 1 (w1|w3 +
 * SwiGLU, or the single-linear GEMM), 1 grouped GEMM phase 2 (w2),
 * 2 compensator t = A U, 3 other.  milo_profile_read returns the number of
 * recorded launches of that kind and their summed duration, then clears. */
void milo_profile_enable(int32_t on);
int64_t milo_profile_read(int32_t kind, double* total_ms);

#ifdef __cplusplus
}
#endif
#endif
