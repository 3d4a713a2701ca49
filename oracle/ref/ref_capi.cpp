// extern "C" surface over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/build_ref.sh).  TEST INFRASTRUCTURE
// ONLY: used by tests/golden/make_golden.py to pin the C restatement in
// oracle/milo_oracle.c, and by bench.py's cpu_baseline / --impl reference leg.
// Never linked into the product library.
//
// Every function here forwards to reference code; the only logic of our own
// is argument marshalling and the MoE composition (the reference has no MoE
// layer): ref_moe_forward composes per-expert
// milo::gemm_w3a16 calls (proj/src/gemm.cpp:117-199) run through the
// reference's own milo::parallel_for (proj/src/pipeline.cpp:26-53).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "milo/errors.hpp"
#include "milo/gemm.hpp"
#include "milo/half.hpp"
#include "milo/lowrank.hpp"
#include "milo/pack.hpp"
#include "milo/pipeline.hpp"
#include "milo/quant.hpp"
#include "milo/rank_policy.hpp"
#include "milo/stats.hpp"
#include "milo/synth.hpp"
#include "milo/tensor_store.hpp"

using namespace milo;

namespace {
thread_local std::string g_err;

int status_of(const MiloError& e) { return static_cast<int>(e.code()) + 1; }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const MiloError& e) {
    g_err = e.what();
    return status_of(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

PackedInt3Matrix make_packed(std::uint64_t rows, std::uint64_t cols, int layout, int split,
                             int mode, std::uint64_t group_size, const std::uint32_t* words,
                             const std::uint32_t* plane_a, const std::uint32_t* plane_b,
                             const std::uint16_t* scales, const std::uint16_t* zeros) {
  PackedInt3Matrix p;
  p.rows = rows;
  p.cols = cols;
  p.layout = layout == 0 ? PackLayout::Linear : PackLayout::Tiled16x64;
  p.split = split != 0;
  p.mode = mode == 0 ? DequantMode::Symmetric : DequantMode::Asymmetric;
  p.group_size = group_size;
  const std::size_t groups = rows * cols / 32;
  if (p.split) {
    p.plane_a.assign(plane_a, plane_a + groups * 2);
    p.plane_b.assign(plane_b, plane_b + groups);
  } else {
    p.words.assign(words, words + groups * 3);
  }
  const std::size_t qg = rows * cols / group_size;
  p.scales.assign(scales, scales + qg);
  if (zeros) p.zeros.assign(zeros, zeros + qg);
  return p;
}

void export_packed(const PackedInt3Matrix& p, std::uint32_t* words, std::uint32_t* plane_a,
                   std::uint32_t* plane_b, std::uint16_t* scales, std::uint16_t* zeros) {
  if (p.split) {
    if (plane_a) std::memcpy(plane_a, p.plane_a.data(), p.plane_a.size() * 4);
    if (plane_b) std::memcpy(plane_b, p.plane_b.data(), p.plane_b.size() * 4);
  } else if (words) {
    std::memcpy(words, p.words.data(), p.words.size() * 4);
  }
  if (scales) std::memcpy(scales, p.scales.data(), p.scales.size() * 2);
  if (zeros && !p.zeros.empty()) std::memcpy(zeros, p.zeros.data(), p.zeros.size() * 2);
}

std::optional<Compensator> make_comp(std::uint64_t rows, std::uint64_t cols, std::uint64_t rank,
                                     int storage, const float* U, const float* V,
                                     const std::uint8_t* qu_codes, const float* qu_scales,
                                     const std::uint8_t* qvt_codes, const float* qvt_scales,
                                     std::uint64_t group_size) {
  Compensator c;
  c.rows = rows;
  c.cols = cols;
  c.rank = rank;
  if (storage == 0) {
    c.storage = CompensatorStorage::Real;
    c.U.assign(U, U + rows * rank);
    c.V.assign(V, V + rank * cols);
  } else {
    c.storage = CompensatorStorage::SymmInt3;
    const std::size_t gpr = rank == 0 ? 0 : (rank + group_size - 1) / group_size;
    c.qU.rows = rows;
    c.qU.cols = rank;
    c.qU.group_size = group_size;
    c.qVt.rows = cols;
    c.qVt.cols = rank;
    c.qVt.group_size = group_size;
    if (rank > 0) {
      c.qU.codes.assign(qu_codes, qu_codes + rows * rank);
      c.qU.scales.assign(qu_scales, qu_scales + rows * gpr);
      c.qVt.codes.assign(qvt_codes, qvt_codes + cols * rank);
      c.qVt.scales.assign(qvt_scales, qvt_scales + cols * gpr);
    }
  }
  return c;
}

GemmConfig make_cfg(int tile_k, int tile_n, std::uint64_t group_size, int mode, int depth,
                    int materialize) {
  GemmConfig cfg;
  cfg.tile_shape = {tile_k, tile_n};
  cfg.group_size = group_size;
  cfg.mode = mode == 0 ? DequantMode::Symmetric : DequantMode::Asymmetric;
  cfg.pipeline_depth = depth;
  cfg.materialize_compensator = materialize != 0;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- half.hpp -----------------------------------------------------------------
std::uint16_t ref_float_to_half(float f) { return float_to_half(f); }
float ref_half_to_float(std::uint16_t h) { return half_to_float(h); }
std::uint16_t ref_double_to_half(double d) { return double_to_half(d); }
std::uint16_t ref_half_add(std::uint16_t a, std::uint16_t b) { return half_add(a, b); }
std::uint16_t ref_half_sub(std::uint16_t a, std::uint16_t b) { return half_sub(a, b); }
std::uint16_t ref_half_mul(std::uint16_t a, std::uint16_t b) { return half_mul(a, b); }
std::uint16_t ref_half_fma(std::uint16_t a, std::uint16_t b, std::uint16_t c) {
  return half_fma(a, b, c);
}

// --- pack.hpp -------------------------------------------------------------------
int ref_pack32(const std::uint8_t* codes, std::uint64_t n, std::uint32_t* out3) {
  return guarded([&] {
    auto w = pack32(std::span<const std::uint8_t>(codes, n));
    std::memcpy(out3, w.data(), 12);
  });
}

void ref_unpack32(const std::uint32_t* w3, std::uint8_t* out32) {
  auto c = unpack32({w3[0], w3[1], w3[2]});
  std::memcpy(out32, c.data(), 32);
}

void ref_fast_dequant_pair(std::uint32_t word, int pair, int mode, std::uint16_t* out2) {
  auto [lo, hi] = fast_dequant_pair(word, pair,
                                    mode == 0 ? DequantMode::Symmetric : DequantMode::Asymmetric);
  out2[0] = lo;
  out2[1] = hi;
}

std::uint16_t ref_symmetric_step(std::uint16_t s) { return symmetric_step(s); }
std::uint16_t ref_asymmetric_offset(std::uint16_t s, std::uint16_t z) {
  return asymmetric_offset(s, z);
}

std::uint64_t ref_tiled_position(std::uint64_t rows, std::uint64_t cols, std::uint64_t i,
                                 std::uint64_t j) {
  return tiled_position(rows, cols, i, j);
}

// Packs logical codes through the reference's own pack_linear /
// pack_linear_symmetric / reshuffle_tiled / split_planes.  zeros == nullptr
// selects symmetric mode.
int ref_pack_matrix(std::uint64_t rows, std::uint64_t cols, const std::uint8_t* codes,
                    const float* scales, const float* zeros, std::uint64_t group_size, int tiled,
                    int split, std::uint32_t* words, std::uint32_t* plane_a,
                    std::uint32_t* plane_b, std::uint16_t* scales_h, std::uint16_t* zeros_h) {
  return guarded([&] {
    PackedInt3Matrix p;
    const std::size_t qg = rows * cols / group_size;
    if (zeros == nullptr) {
      std::vector<std::uint8_t> c(codes, codes + rows * cols);
      std::vector<float> s(scales, scales + qg);
      p = pack_linear_symmetric(rows, cols, c, s, group_size);
      if (tiled) throw ConfigError("reference reshuffle_tiled is asymmetric-only");
    } else {
      QuantizedMatrix q;
      q.rows = rows;
      q.cols = cols;
      q.bits = 3;
      q.group_size = group_size;
      q.codes.assign(codes, codes + rows * cols);
      q.scales.assign(scales, scales + qg);
      q.zeros.assign(zeros, zeros + qg);
      p = tiled ? reshuffle_tiled(q) : pack_linear(q);
    }
    if (split) p = split_planes(p);
    export_packed(p, words, plane_a, plane_b, scales_h, zeros_h);
  });
}

int ref_unpack_codes(std::uint64_t rows, std::uint64_t cols, int layout, int split, int mode,
                     std::uint64_t group_size, const std::uint32_t* words,
                     const std::uint32_t* plane_a, const std::uint32_t* plane_b,
                     const std::uint16_t* scales, const std::uint16_t* zeros,
                     std::uint8_t* out) {
  return guarded([&] {
    PackedInt3Matrix p = make_packed(rows, cols, layout, split, mode, group_size, words, plane_a,
                                     plane_b, scales, zeros);
    auto c = unpack_codes(p);
    std::memcpy(out, c.data(), c.size());
  });
}

// The reference's own packed-i3 container writer / reader (pack.cpp:306-400):
// test fixtures for milo_weight_load come from save_packed, and load_packed is
// the parity reference for the B200 library's reader.
int ref_save_packed(std::uint64_t rows, std::uint64_t cols, int layout, int split, int mode,
                    std::uint64_t group_size, const std::uint32_t* words,
                    const std::uint32_t* plane_a, const std::uint32_t* plane_b,
                    const std::uint16_t* scales, const std::uint16_t* zeros, const char* name,
                    const char* path) {
  return guarded([&] {
    PackedInt3Matrix p = make_packed(rows, cols, layout, split, mode, group_size, words, plane_a,
                                     plane_b, scales, zeros);
    save_packed(p, name, path);
  });
}

// Header fields of a packed-i3 container (load_packed); out6 = rows, cols, layout,
// split, mode, group_size.
int ref_load_packed_info(const char* path, std::uint64_t* out6) {
  return guarded([&] {
    PackedInt3Matrix p = load_packed(path);
    out6[0] = p.rows;
    out6[1] = p.cols;
    out6[2] = p.layout == PackLayout::Linear ? 0 : 1;
    out6[3] = p.split ? 1 : 0;
    out6[4] = p.mode == DequantMode::Symmetric ? 0 : 1;
    out6[5] = p.group_size;
  });
}

// Payload of a packed-i3 container (load_packed) into caller buffers sized from the info.
int ref_load_packed(const char* path, std::uint32_t* words, std::uint32_t* plane_a,
                    std::uint32_t* plane_b, std::uint16_t* scales, std::uint16_t* zeros) {
  return guarded([&] {
    PackedInt3Matrix p = load_packed(path);
    export_packed(p, words, plane_a, plane_b, scales, zeros);
  });
}

int ref_dequant_packed_half(std::uint64_t rows, std::uint64_t cols, int layout, int split,
                            int mode, std::uint64_t group_size, const std::uint32_t* words,
                            const std::uint32_t* plane_a, const std::uint32_t* plane_b,
                            const std::uint16_t* scales, const std::uint16_t* zeros,
                            int dq_mode, std::uint16_t* out) {
  return guarded([&] {
    PackedInt3Matrix p = make_packed(rows, cols, layout, split, mode, group_size, words, plane_a,
                                     plane_b, scales, zeros);
    auto h = dequant_packed_half(p, dq_mode == 0 ? DequantMode::Symmetric
                                                 : DequantMode::Asymmetric);
    std::memcpy(out, h.data(), h.size() * 2);
  });
}

// --- quant.hpp (grouped min/max quantizer, used to make synthetic weights) --------
int ref_quantize_minmax(std::uint64_t rows, std::uint64_t cols, const float* w,
                        std::uint8_t* codes, float* scales, float* zeros) {
  return guarded([&] {
    WeightMatrix m(rows, cols);
    std::memcpy(m.data.data(), w, rows * cols * 4);
    QuantConfig qc;
    QuantParams params = init_quant_params(m, qc);
    QuantizedMatrix q = quantize(m, params.scales, params.zeros, qc);
    std::memcpy(codes, q.codes.data(), q.codes.size());
    std::memcpy(scales, q.scales.data(), q.scales.size() * 4);
    std::memcpy(zeros, q.zeros.data(), q.zeros.size() * 4);
  });
}

// Mirrors pipeline.cpp:408-426 random_packed (anonymous in the reference):
// the seeded synthetic weights gemm-check runs on.  Outputs linear layout.
int ref_random_packed(std::uint64_t k, std::uint64_t n, int mode, std::uint64_t seed,
                      std::uint32_t* words, std::uint16_t* scales_h, std::uint16_t* zeros_h) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    PackedInt3Matrix p;
    if (mode == 1) {
      WeightMatrix w(k, n);
      std::normal_distribution<float> dist(0.0f, 0.05f);
      for (float& v : w.data) v = dist(rng);
      QuantConfig qc;
      QuantParams params = init_quant_params(w, qc);
      p = pack_linear(quantize(w, params.scales, params.zeros, qc));
    } else {
      std::vector<std::uint8_t> codes(k * n);
      std::uniform_int_distribution<int> cdist(0, 7);
      for (auto& c : codes) c = static_cast<std::uint8_t>(cdist(rng));
      std::vector<float> scales(k * n / 64);
      std::normal_distribution<float> sdist(0.0f, 0.05f);
      for (float& s : scales) s = std::fabs(sdist(rng)) + 0.01f;
      p = pack_linear_symmetric(k, n, codes, scales, 64);
    }
    export_packed(p, words, nullptr, nullptr, scales_h, zeros_h);
  });
}

// libstdc++ N(mean, sigma) stream with the reference's engine (mt19937_64);
// the reference's generators all use this pairing (pipeline.cpp:544-547).
void ref_fill_normal(std::uint64_t seed, std::uint64_t count, float mean, float sigma,
                     float* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<float> dist(mean, sigma);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = dist(rng);
}

std::uint64_t ref_fnv1a64(const char* s) { return fnv1a64(s); }

// --- lowrank.hpp ----------------------------------------------------------------
int ref_symm_int3_quantize(const float* values, std::uint64_t rows, std::uint64_t cols,
                           std::uint64_t group_size, std::uint8_t* codes, float* scales) {
  return guarded([&] {
    std::vector<float> v(values, values + rows * cols);
    SymmInt3Factor f = symm_int3_quantize(v, rows, cols, group_size);
    std::memcpy(codes, f.codes.data(), f.codes.size());
    std::memcpy(scales, f.scales.data(), f.scales.size() * 4);
  });
}

int ref_symm_int3_dequantize(std::uint64_t rows, std::uint64_t cols, std::uint64_t group_size,
                             const std::uint8_t* codes, const float* scales, float* out) {
  return guarded([&] {
    SymmInt3Factor f;
    f.rows = rows;
    f.cols = cols;
    f.group_size = group_size;
    const std::size_t gpr = (cols + group_size - 1) / group_size;
    f.codes.assign(codes, codes + rows * cols);
    f.scales.assign(scales, scales + rows * gpr);
    auto o = symm_int3_dequantize(f);
    std::memcpy(out, o.data(), o.size() * 4);
  });
}

// Compensator::quantize_symm_int3 (lowrank.cpp:34-50) from real factors.
int ref_comp_quantize(std::uint64_t rows, std::uint64_t cols, std::uint64_t rank, const float* U,
                      const float* V, std::uint64_t group_size, std::uint8_t* qu_codes,
                      float* qu_scales, std::uint8_t* qvt_codes, float* qvt_scales) {
  return guarded([&] {
    Compensator c;
    c.rows = rows;
    c.cols = cols;
    c.rank = rank;
    c.U.assign(U, U + rows * rank);
    c.V.assign(V, V + rank * cols);
    c.quantize_symm_int3(group_size);
    if (rank == 0) return;
    std::memcpy(qu_codes, c.qU.codes.data(), c.qU.codes.size());
    std::memcpy(qu_scales, c.qU.scales.data(), c.qU.scales.size() * 4);
    std::memcpy(qvt_codes, c.qVt.codes.data(), c.qVt.codes.size());
    std::memcpy(qvt_scales, c.qVt.scales.data(), c.qVt.scales.size() * 4);
  });
}

// --- gemm.hpp -------------------------------------------------------------------
int ref_gemm_w3a16(const float* A, std::uint64_t m, std::uint64_t rows, std::uint64_t cols,
                   int layout, int split, int mode, std::uint64_t group_size,
                   const std::uint32_t* words, const std::uint32_t* plane_a,
                   const std::uint32_t* plane_b, const std::uint16_t* scales,
                   const std::uint16_t* zeros, int has_comp, std::uint64_t comp_rows,
                   std::uint64_t comp_cols, std::uint64_t rank, int storage, const float* U,
                   const float* V, const std::uint8_t* qu_codes, const float* qu_scales,
                   const std::uint8_t* qvt_codes, const float* qvt_scales,
                   std::uint64_t comp_group, int tile_k, int tile_n, std::uint64_t cfg_group,
                   int cfg_mode, int depth, int materialize, std::uint64_t a_cols, float* C) {
  return guarded([&] {
    PackedInt3Matrix p = make_packed(rows, cols, layout, split, mode, group_size, words, plane_a,
                                     plane_b, scales, zeros);
    WeightMatrix a(m, a_cols);
    std::memcpy(a.data.data(), A, m * a_cols * 4);
    std::optional<Compensator> comp;
    if (has_comp)
      comp = make_comp(comp_rows, comp_cols, rank, storage, U, V, qu_codes, qu_scales, qvt_codes,
                       qvt_scales, comp_group);
    GemmConfig cfg = make_cfg(tile_k, tile_n, cfg_group, cfg_mode, depth, materialize);
    WeightMatrix c = gemm_w3a16(a, p, comp, cfg);
    std::memcpy(C, c.data.data(), c.data.size() * 4);
  });
}

int ref_pipeline_tail_check(std::uint64_t k, int tile_k, int tile_n, int depth, int* stages,
                            int max_stages, int* n_stages) {
  return guarded([&] {
    GemmConfig cfg = make_cfg(tile_k, tile_n, 64, 1, depth, 0);
    TileSchedule s = pipeline_tail_check(k, cfg);
    *n_stages = static_cast<int>(s.stage_tiles.size());
    for (int i = 0; i < *n_stages && i < max_stages; ++i) stages[i] = s.stage_tiles[i];
  });
}

std::uint64_t ref_matrix_memory_bytes(std::uint64_t rows, std::uint64_t cols, std::uint64_t rank,
                                      int bits, std::uint64_t group_size, int comp_bits) {
  try {
    return matrix_memory_bytes(rows, cols, rank, bits, group_size, comp_bits);
  } catch (const MiloError& e) {
    g_err = e.what();
    return 0;
  }
}

// --- MoE composition over the reference GEMM (CPU baseline) -----------------------
// One expert = w1 (d x f), w3 (d x f), w2 (f x d) in the reference's k x n
// orientation (synth.cpp:37-39), each a linear PackedInt3Matrix with an optional
// symm-int3 compensator.  Routing is given (topk ids/weights per token).
//
// Threading: the reference's gemm_w3a16 is single-threaded; its output columns
// are independent (C[i,j] accumulates over k in a fixed order per column, and
// the compensator adds t V[:, j] per column), so every matrix is cut once into
// column slices (multiples of 128: whole quant groups and whole n-tiles of the
// GemmConfig tile (128,128), gemm.cpp:131-134) and the calls of a
// phase -- (touched expert, w1 | w3, slice), then (touched expert, w2, slice) --
// run through the reference's own milo::parallel_for (pipeline.cpp:26-53) over
// all workers.  The result is bit-identical to the unsliced composition.
struct RefLinear {
  PackedInt3Matrix w;
  std::optional<Compensator> comp;
  // column slices (built on first use for a slice count)
  std::size_t n_slices = 0;
  std::vector<std::size_t> c0;  // first column of each slice (+ end)
  std::vector<PackedInt3Matrix> ws;
  std::vector<std::optional<Compensator>> cs;
};
struct RefExpert {
  RefLinear l[3];  // w1, w3, w2
};

// Columns [a, b) of a linear-layout, non-split packed matrix (a, b multiples of 128).
PackedInt3Matrix slice_cols(const PackedInt3Matrix& p, std::size_t a, std::size_t b) {
  PackedInt3Matrix q;
  q.rows = p.rows;
  q.cols = b - a;
  q.layout = p.layout;
  q.split = false;
  q.mode = p.mode;
  q.group_size = p.group_size;
  const std::size_t gpr = p.cols / 32, qpr = p.cols / p.group_size;
  q.words.reserve(p.rows * (b - a) / 32 * 3);
  q.scales.reserve(p.rows * (b - a) / p.group_size);
  for (std::size_t r = 0; r < p.rows; ++r) {
    q.words.insert(q.words.end(), p.words.begin() + (r * gpr + a / 32) * 3,
                   p.words.begin() + (r * gpr + b / 32) * 3);
    q.scales.insert(q.scales.end(), p.scales.begin() + r * qpr + a / p.group_size,
                    p.scales.begin() + r * qpr + b / p.group_size);
    if (!p.zeros.empty())
      q.zeros.insert(q.zeros.end(), p.zeros.begin() + r * qpr + a / p.group_size,
                     p.zeros.begin() + r * qpr + b / p.group_size);
  }
  return q;
}

// Columns [a, b) of a compensator: U unchanged, V^T rows [a, b).
std::optional<Compensator> slice_comp(const std::optional<Compensator>& c, std::size_t a, std::size_t b) {
  if (!c) return std::nullopt;
  Compensator s = *c;
  s.cols = b - a;
  if (c->storage == CompensatorStorage::Real) {
    s.V.clear();
    for (std::size_t r = 0; r < c->rank; ++r)
      s.V.insert(s.V.end(), c->V.begin() + r * c->cols + a, c->V.begin() + r * c->cols + b);
  } else {
    const std::size_t gpr = c->rank == 0 ? 0 : (c->rank + c->qVt.group_size - 1) / c->qVt.group_size;
    s.qVt.rows = b - a;
    s.qVt.codes.assign(c->qVt.codes.begin() + a * c->rank, c->qVt.codes.begin() + b * c->rank);
    s.qVt.scales.assign(c->qVt.scales.begin() + a * gpr, c->qVt.scales.begin() + b * gpr);
  }
  return s;
}

void ensure_slices(RefLinear& L, std::size_t want) {
  const std::size_t groups = L.w.cols / 128;
  const std::size_t n = std::max<std::size_t>(1, std::min(want, groups));
  if (L.n_slices == n) return;
  L.n_slices = n;
  L.c0.assign(n + 1, 0);
  L.ws.clear();
  L.cs.clear();
  for (std::size_t s = 0; s <= n; ++s) L.c0[s] = groups * s / n * 128;
  for (std::size_t s = 0; s < n; ++s) {
    if (n == 1) {
      L.ws.push_back(L.w);
      L.cs.push_back(L.comp);
    } else {
      L.ws.push_back(slice_cols(L.w, L.c0[s], L.c0[s + 1]));
      L.cs.push_back(slice_comp(L.comp, L.c0[s], L.c0[s + 1]));
    }
  }
}

void* ref_moe_create(int n_experts) {
  auto* v = new std::vector<RefExpert>(static_cast<std::size_t>(n_experts));
  return v;
}

void ref_moe_destroy(void* h) { delete static_cast<std::vector<RefExpert>*>(h); }

int ref_moe_set_linear(void* h, int expert, int which, std::uint64_t rows, std::uint64_t cols,
                       const std::uint32_t* words, const std::uint16_t* scales,
                       const std::uint16_t* zeros, std::uint64_t rank,
                       const std::uint8_t* qu_codes, const float* qu_scales,
                       const std::uint8_t* qvt_codes, const float* qvt_scales) {
  return guarded([&] {
    auto& ex = (*static_cast<std::vector<RefExpert>*>(h))[static_cast<std::size_t>(expert)];
    RefLinear& L = ex.l[which];
    L = RefLinear{};
    L.w = make_packed(rows, cols, 0, 0, zeros ? 1 : 0, 64, words, nullptr, nullptr, scales, zeros);
    if (rank > 0)
      L.comp = make_comp(rows, cols, rank, 1, nullptr, nullptr, qu_codes, qu_scales, qvt_codes,
                         qvt_scales, 64);
    else
      L.comp.reset();
  });
}

// Prepares the column slices for `workers` threads (outside any timed region).
int ref_moe_prepare(void* h, int workers) {
  return guarded([&] {
    for (auto& ex : *static_cast<std::vector<RefExpert>*>(h))
      for (auto& L : ex.l)
        if (L.w.cols) ensure_slices(L, static_cast<std::size_t>(std::max(1, workers)));
  });
}

// x: m x d fp32; topk_ids/topk_w: m x K; out: m x d fp32.  shared experts
// (ids >= n_routed) are applied to every token with weight 1 by the caller
// encoding them in topk lists, so this function is routing-agnostic.
int ref_moe_forward(void* h, const float* x, std::uint64_t m, std::uint64_t d, int K,
                    const std::int32_t* topk_ids, const float* topk_w, int workers, float* out) {
  return guarded([&] {
    auto& experts = *static_cast<std::vector<RefExpert>*>(h);
    const std::size_t E = experts.size();
    std::vector<std::vector<std::size_t>> rows_of(E);
    for (std::size_t t = 0; t < m; ++t)
      for (int k = 0; k < K; ++k) {
        const int e = topk_ids[t * static_cast<std::size_t>(K) + static_cast<std::size_t>(k)];
        if (e >= 0) rows_of[static_cast<std::size_t>(e)].push_back(t);
      }
    std::vector<std::size_t> active;
    for (std::size_t e = 0; e < E; ++e)
      if (!rows_of[e].empty()) active.push_back(e);
    const std::size_t want = static_cast<std::size_t>(std::max(1, workers));
    for (std::size_t e : active)
      for (auto& L : experts[e].l) ensure_slices(L, want);
    GemmConfig cfg;
    cfg.tile_shape = {128, 128};
    // gathered rows of every touched expert
    std::vector<WeightMatrix> xe(E), h1(E), h3(E), y(E);
    for (std::size_t e : active) {
      const auto& rows = rows_of[e];
      xe[e] = WeightMatrix(rows.size(), d);
      for (std::size_t i = 0; i < rows.size(); ++i)
        std::memcpy(&xe[e].data[i * d], x + rows[i] * d, d * 4);
      const std::size_t f = experts[e].l[0].w.cols;
      h1[e] = WeightMatrix(rows.size(), f);
      h3[e] = WeightMatrix(rows.size(), f);
      y[e] = WeightMatrix(rows.size(), d);
    }
    auto run_slice = [&](const RefLinear& L, std::size_t s, const WeightMatrix& a, WeightMatrix& c) {
      const WeightMatrix part = gemm_w3a16(a, L.ws[s], L.cs[s], cfg);
      const std::size_t w = L.c0[s + 1] - L.c0[s];
      for (std::size_t i = 0; i < a.rows; ++i)
        std::memcpy(&c.data[i * c.cols + L.c0[s]], &part.data[i * w], w * 4);
    };
    // phase 1: (expert, w1 | w3, slice)
    std::vector<std::array<std::size_t, 3>> jobs;
    for (std::size_t e : active)
      for (std::size_t j = 0; j < 2; ++j)
        for (std::size_t s = 0; s < experts[e].l[j].n_slices; ++s) jobs.push_back({e, j, s});
    parallel_for(jobs.size(), workers, [&](std::size_t i) {
      const auto [e, j, s] = jobs[i];
      run_slice(experts[e].l[j], s, xe[e], j == 0 ? h1[e] : h3[e]);
    });
    for (std::size_t e : active)
      for (std::size_t i = 0; i < h1[e].data.size(); ++i) {
        const float a = h1[e].data[i];
        h1[e].data[i] = a / (1.0f + std::exp(-a)) * h3[e].data[i];
      }
    // phase 2: (expert, w2, slice)
    jobs.clear();
    for (std::size_t e : active)
      for (std::size_t s = 0; s < experts[e].l[2].n_slices; ++s) jobs.push_back({e, 2, s});
    parallel_for(jobs.size(), workers, [&](std::size_t i) {
      const auto [e, j, s] = jobs[i];
      run_slice(experts[e].l[2], s, h1[e], y[e]);
    });
    std::vector<std::size_t> cursor(E, 0);
    std::fill(out, out + m * d, 0.0f);
    for (std::size_t t = 0; t < m; ++t)
      for (int k = 0; k < K; ++k) {
        const int e = topk_ids[t * static_cast<std::size_t>(K) + static_cast<std::size_t>(k)];
        if (e < 0) continue;
        const float w = topk_w[t * static_cast<std::size_t>(K) + static_cast<std::size_t>(k)];
        // rows_of[e] is ascending in t, so the row of token t is found by a cursor.
        const std::size_t r = cursor[static_cast<std::size_t>(e)]++;
        const float* yr = &y[static_cast<std::size_t>(e)].data[r * d];
        for (std::size_t j = 0; j < d; ++j) out[t * d + j] += w * yr[j];
      }
  });
}

// A rank plan by the reference's own pipeline pieces, for a one-layer model of
// `experts` routed experts (layer0.expert<x>.w1|w2|w3, synth.cpp:32-48) plus `shared`
// shared experts (layer0.shared_expert<s>.*, StructureTag::SharedExpert): per-matrix
// kurtosis (stats.cpp) of the reference's synthetic StudentTMix weights
// (synth_matrix, df_min = 5: heavier tails for higher expert indices), then
// plan_ranks(manifest, stats, parse_policy(policy)) (rank_policy.cpp:94-164).  Weights
// are synthesized at stats_rows x stats_cols (their per-expert distribution does not
// depend on the shape; 0 = the model's shape).  ranks: (experts + shared) x 3 in
// w1, w3, w2 order; kurt: experts x 3.  Returns 0, or the ErrorCode + 1.
int ref_plan_synth(int experts, int shared, std::uint64_t model_dim, std::uint64_t ffn_dim,
                   std::uint64_t stats_rows, std::uint64_t stats_cols, std::uint64_t seed,
                   const char* policy, int32_t* ranks, double* kurt) {
  return guarded([&] {
    SynthSpec spec;
    spec.layers = 1;
    spec.experts = experts;
    spec.model_dim = model_dim;
    spec.ffn_dim = ffn_dim;
    spec.seed = seed;
    spec.expert_dist = ExpertDist::StudentTMix;
    spec.expert_df_min = 5.0;
    ModelManifest man = synth_manifest(spec);
    for (int s = 0; s < shared; ++s)
      for (const char* w : {"w1", "w2", "w3"}) {
        MatrixEntry e;
        e.name = "layer0.shared_expert" + std::to_string(s) + "." + w;
        e.rows = std::string(w) == "w2" ? ffn_dim : model_dim;
        e.cols = std::string(w) == "w2" ? model_dim : ffn_dim;
        e.structure_tag = StructureTag::SharedExpert;
        man.layers[0].matrices.push_back(e);
      }
    std::vector<const MatrixEntry*> exp;
    for (const MatrixEntry* e : man.all_matrices())
      if (e->structure_tag == StructureTag::Expert) exp.push_back(e);
    std::vector<double> k(exp.size());
    std::vector<std::thread> pool;
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (std::size_t i = t; i < exp.size(); i += nt) {
          MatrixEntry e = *exp[i];
          if (stats_rows) {
            e.rows = stats_rows;
            e.cols = stats_cols;
          }
          k[i] = kurtosis(synth_matrix(spec, e));
        }
      });
    for (auto& th : pool) th.join();
    std::map<std::string, MatrixStats> stats;
    for (std::size_t i = 0; i < exp.size(); ++i) {
      MatrixStats s;
      s.name = exp[i]->name;
      s.kurtosis = k[i];
      s.structure_tag = StructureTag::Expert;
      stats[s.name] = s;
    }
    const RankPlan plan = plan_ranks(man, stats, parse_policy(policy));
    const char* order[3] = {"w1", "w3", "w2"};
    for (int x = 0; x < experts + shared; ++x)
      for (int j = 0; j < 3; ++j) {
        const std::string name = x < experts ? "layer0.expert" + std::to_string(x) + "." + order[j]
                                             : "layer0.shared_expert" + std::to_string(x - experts) + "." + order[j];
        ranks[x * 3 + j] = static_cast<int32_t>(plan.ranks.at(name));
        if (x < experts)
          for (std::size_t i = 0; i < exp.size(); ++i)
            if (exp[i]->name == name) kurt[x * 3 + j] = k[i];
      }
  });
}

}  // extern "C"
