// milo_b200.hpp — header-only C++ host API over the C ABI (milo_b200.h),
// mirroring the reference's operator types so a caller of
//
//   milo::gemm_w3a16(const WeightMatrix&, const PackedInt3Matrix&,
//                    const std::optional<Compensator>&, const GemmConfig&)
//   (/root/reference/proj/include/milo/gemm.hpp:43-48)
//
// switches by replacing the packed weight / compensator with their device
// handles.  Errors are thrown as milo::b200::MiloError subclasses carrying the
// reference's ErrorCode categories (errors.hpp:9-48).
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "milo_b200.h"

namespace milo::b200 {

// ---- errors (errors.hpp:9-48) ------------------------------------------------
enum class ErrorCode { Format, Data, Io, Shape, Rank, Numeric, Stat, Plan, Range, Config, Cuda, Argument };

class MiloError : public std::runtime_error {
 public:
  MiloError(ErrorCode c, const std::string& m) : std::runtime_error(m), code_(c) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

#define MILO_B200_ERROR(Name, Code) \
  class Name : public MiloError {   \
   public:                          \
    explicit Name(const std::string& m) : MiloError(ErrorCode::Code, m) {} \
  }
MILO_B200_ERROR(FormatError, Format);
MILO_B200_ERROR(DataError, Data);
MILO_B200_ERROR(IoError, Io);
MILO_B200_ERROR(ShapeError, Shape);
MILO_B200_ERROR(RankError, Rank);
MILO_B200_ERROR(NumericError, Numeric);
MILO_B200_ERROR(StatError, Stat);
MILO_B200_ERROR(PlanError, Plan);
MILO_B200_ERROR(RangeError, Range);
MILO_B200_ERROR(ConfigError, Config);
MILO_B200_ERROR(CudaError, Cuda);
MILO_B200_ERROR(ArgumentError, Argument);
#undef MILO_B200_ERROR

inline void check(milo_status s) {
  if (s == MILO_OK) return;
  const std::string m = milo_last_error();
  switch (s) {
    case MILO_ERR_FORMAT: throw FormatError(m);
    case MILO_ERR_DATA: throw DataError(m);
    case MILO_ERR_IO: throw IoError(m);
    case MILO_ERR_SHAPE: throw ShapeError(m);
    case MILO_ERR_RANK: throw RankError(m);
    case MILO_ERR_NUMERIC: throw NumericError(m);
    case MILO_ERR_STAT: throw StatError(m);
    case MILO_ERR_PLAN: throw PlanError(m);
    case MILO_ERR_RANGE: throw RangeError(m);
    case MILO_ERR_CONFIG: throw ConfigError(m);
    case MILO_ERR_CUDA: throw CudaError(m);
    default: throw ArgumentError(m);
  }
}

// ---- value types mirroring the reference -------------------------------------
enum class PackLayout { Linear = 0, Tiled16x64 = 1 };          // pack.hpp:37
enum class DequantMode { Symmetric = 0, Asymmetric = 1 };      // pack.hpp:38
enum class CompensatorStorage { Real = 0, SymmInt3 = 1 };      // lowrank.hpp:13

struct WeightMatrix {  // matrix.hpp:14-37
  std::size_t rows = 0, cols = 0;
  std::vector<float> data;
  std::string name;
  WeightMatrix() = default;
  WeightMatrix(std::size_t r, std::size_t c, std::string n = {})
      : rows(r), cols(c), data(r * c, 0.0f), name(std::move(n)) {}
};

struct PackedInt3Matrix {  // pack.hpp:45-66
  std::size_t rows = 0, cols = 0;
  PackLayout layout = PackLayout::Linear;
  bool split = false;
  DequantMode mode = DequantMode::Asymmetric;
  std::size_t group_size = 64;
  std::vector<std::uint32_t> words, plane_a, plane_b;
  std::vector<std::uint16_t> scales, zeros;
};

struct SymmInt3Factor {  // lowrank.hpp:19-25
  std::size_t rows = 0, cols = 0, group_size = 64;
  std::vector<std::uint8_t> codes;
  std::vector<float> scales;
};

struct Compensator {  // lowrank.hpp:31-50
  std::size_t rows = 0, cols = 0, rank = 0;
  CompensatorStorage storage = CompensatorStorage::Real;
  std::vector<float> U, V;
  SymmInt3Factor qU, qVt;
};

struct GemmConfig {  // gemm.hpp:17-25
  std::pair<int, int> tile_shape{128, 128};
  std::size_t group_size = 64;
  DequantMode mode = DequantMode::Asymmetric;
  int pipeline_depth = 4;
  bool materialize_compensator = false;

  milo_gemm_config c() const {
    return {tile_shape.first, tile_shape.second, group_size, static_cast<int32_t>(mode),
            pipeline_depth, materialize_compensator ? 1 : 0};
  }
};

// ---- device handles ---------------------------------------------------------------
class DeviceWeight {
 public:
  explicit DeviceWeight(const PackedInt3Matrix& p) {
    milo_packed_desc d{};
    d.rows = p.rows;
    d.cols = p.cols;
    d.layout = static_cast<int32_t>(p.layout);
    d.split = p.split ? 1 : 0;
    d.mode = static_cast<int32_t>(p.mode);
    d.group_size = p.group_size;
    d.words = p.words.empty() ? nullptr : p.words.data();
    d.n_words = p.words.size();
    d.plane_a = p.plane_a.empty() ? nullptr : p.plane_a.data();
    d.n_plane_a = p.plane_a.size();
    d.plane_b = p.plane_b.empty() ? nullptr : p.plane_b.data();
    d.n_plane_b = p.plane_b.size();
    d.scales = p.scales.empty() ? nullptr : p.scales.data();
    d.n_scales = p.scales.size();
    d.zeros = p.zeros.empty() ? nullptr : p.zeros.data();
    d.n_zeros = p.zeros.size();
    milo_weight* w = nullptr;
    check(milo_weight_create(&d, &w));
    h_.reset(w);
  }
  // From a packed-i3 MILO1 container (milo::load_packed, pack.cpp:345-400): the
  // artifacts `milo quantize` / `milo pack` write (pipeline.cpp:324,398).
  static DeviceWeight load(const std::string& path) {
    milo_weight* w = nullptr;
    check(milo_weight_load(path.c_str(), &w));
    return DeviceWeight(w);
  }
  const milo_weight* get() const { return h_.get(); }
  std::size_t rows() const { return info().first; }
  std::size_t cols() const { return info().second; }

 private:
  explicit DeviceWeight(milo_weight* w) { h_.reset(w); }
  std::pair<std::size_t, std::size_t> info() const {
    uint64_t r = 0, c = 0;
    check(milo_weight_info(h_.get(), &r, &c, nullptr, nullptr));
    return {r, c};
  }
  struct Del {
    void operator()(milo_weight* w) const { milo_weight_destroy(w); }
  };
  std::unique_ptr<milo_weight, Del> h_;
};

class DeviceCompensator {
 public:
  explicit DeviceCompensator(const Compensator& c) {
    milo_comp_desc d{};
    d.rows = c.rows;
    d.cols = c.cols;
    d.rank = c.rank;
    d.storage = static_cast<int32_t>(c.storage);
    d.U = c.U.empty() ? nullptr : c.U.data();
    d.V = c.V.empty() ? nullptr : c.V.data();
    d.qu_codes = c.qU.codes.empty() ? nullptr : c.qU.codes.data();
    d.qu_scales = c.qU.scales.empty() ? nullptr : c.qU.scales.data();
    d.qvt_codes = c.qVt.codes.empty() ? nullptr : c.qVt.codes.data();
    d.qvt_scales = c.qVt.scales.empty() ? nullptr : c.qVt.scales.data();
    d.group_size = c.qU.group_size;
    milo_comp* h = nullptr;
    check(milo_comp_create(&d, &h));
    h_.reset(h);
  }
  // From the factor pair `milo quantize` writes (<name>.u.milo / <name>.v.milo,
  // pipeline.cpp:233-283).
  static DeviceCompensator load(const std::string& u_path, const std::string& v_path) {
    milo_comp* h = nullptr;
    check(milo_comp_load(u_path.c_str(), v_path.c_str(), &h));
    return DeviceCompensator(h);
  }
  const milo_comp* get() const { return h_.get(); }
  std::size_t rank() const {
    uint64_t r = 0;
    check(milo_comp_info(h_.get(), nullptr, nullptr, &r, nullptr));
    return r;
  }

 private:
  explicit DeviceCompensator(milo_comp* h) { h_.reset(h); }
  struct Del {
    void operator()(milo_comp* c) const { milo_comp_destroy(c); }
  };
  std::unique_ptr<milo_comp, Del> h_;
};

// ---- the operator ------------------------------------------------------------------
// Host-buffer form: same signature shape and by-value result as the reference.
inline WeightMatrix gemm_w3a16(const WeightMatrix& A, const DeviceWeight& Wp,
                               const DeviceCompensator* comp, const GemmConfig& cfg) {
  const milo_gemm_config c = cfg.c();
  WeightMatrix out(A.rows, Wp.cols(), A.name);
  check(milo_gemm_w3a16_host(Wp.get(), comp ? comp->get() : nullptr, &c, A.data.data(),
                             static_cast<int64_t>(A.rows), static_cast<int64_t>(A.cols),
                             out.data.data()));
  return out;
}

// Device-pointer, stream-ordered form.
inline void gemm_w3a16(const void* A, int64_t m, int64_t a_cols, milo_dtype a_dtype,
                       const DeviceWeight& Wp, const DeviceCompensator* comp,
                       const GemmConfig& cfg, void* C, milo_dtype c_dtype, void* stream) {
  const milo_gemm_config c = cfg.c();
  check(milo_gemm_w3a16(Wp.get(), comp ? comp->get() : nullptr, &c, A, m, a_cols, a_dtype, C,
                        c_dtype, stream));
}

// ---- the top-k routed grouped-expert layer (new) ---------------------------------
struct ExpertRef {
  const DeviceWeight* w1;
  const DeviceWeight* w3;
  const DeviceWeight* w2;
  const DeviceCompensator* c1 = nullptr;
  const DeviceCompensator* c3 = nullptr;
  const DeviceCompensator* c2 = nullptr;
};

class MoELayer {
 public:
  MoELayer(const std::vector<ExpertRef>& experts, const std::vector<ExpertRef>& shared, int top_k,
           milo_score_mode score_mode = MILO_SCORE_SOFTMAX_TOPK) {
    auto conv = [](const std::vector<ExpertRef>& v) {
      std::vector<milo_expert_desc> d;
      for (const auto& e : v)
        d.push_back({e.w1->get(), e.w3->get(), e.w2->get(), e.c1 ? e.c1->get() : nullptr,
                     e.c3 ? e.c3->get() : nullptr, e.c2 ? e.c2->get() : nullptr});
      return d;
    };
    auto de = conv(experts), ds = conv(shared);
    milo_moe* h = nullptr;
    check(milo_moe_create(de.data(), static_cast<int32_t>(de.size()), ds.data(),
                          static_cast<int32_t>(ds.size()), top_k, score_mode, &h));
    h_.reset(h);
  }
  // Host buffers: x (m x d), router logits (m x E) -> out (m x d).
  WeightMatrix forward(const WeightMatrix& x, const WeightMatrix& router_logits) const {
    WeightMatrix out(x.rows, x.cols);
    if (router_logits.rows != x.rows) throw ShapeError("router logits rows != x rows");
    check(milo_moe_forward_host(h_.get(), x.data.data(), static_cast<int64_t>(x.rows),
                                static_cast<int64_t>(x.cols), router_logits.data.data(),
                                static_cast<int64_t>(router_logits.cols), out.data.data()));
    return out;
  }
  // The router gate (E x d binary16 bits, host), then forward_x routes from x itself.
  void set_gate(const std::vector<std::uint16_t>& gate, int64_t n_experts, int64_t d) {
    if (gate.size() != static_cast<std::size_t>(n_experts * d)) throw ShapeError("gate size != E * d");
    check(milo_moe_set_gate(h_.get(), gate.data(), n_experts, d));
  }
  // Device buffers, stream-ordered: router GEMM -> top-k -> experts -> combine.
  void forward_x(const void* x, int64_t m, milo_dtype x_dtype, void* out, milo_dtype out_dtype,
                 void* stream) const {
    check(milo_moe_forward_x(h_.get(), x, m, x_dtype, out, out_dtype, nullptr, nullptr, stream));
  }
  // Device buffers, stream-ordered.
  void forward(const void* x, int64_t m, milo_dtype x_dtype, const float* logits, void* out,
               milo_dtype out_dtype, void* stream) const {
    check(milo_moe_forward(h_.get(), x, m, x_dtype, logits, out, out_dtype, nullptr, nullptr,
                           stream));
  }

 private:
  struct Del {
    void operator()(milo_moe* m) const { milo_moe_destroy(m); }
  };
  std::unique_ptr<milo_moe, Del> h_;
};

}  // namespace milo::b200
