// The INTEGRATION.md section 2 binding, compiled: the reference's own types and
// gemm_w3a16 (the compiled, unmodified reference in oracle/_ref) next to the B200
// library called through include/milo_b200.hpp via field-by-field `to_b200` copies --
// the change a maintainer makes in run_gemm_check (/root/reference/proj/src/
// pipeline.cpp:541-577): upload the packed matrix once, then call the device GEMM with
// the same arguments and compare rows like rel_error_rows.  Built by oracle/build_ref.sh
// into oracle/_ref/b200_binding_check (test infrastructure; needs the reference sources
// at build time only); run by tests/test_gpu_cpp_api.py on a GPU.
#include <cmath>
#include <cstdio>
#include <optional>
#include <random>
#include <vector>

#include "milo/gemm.hpp"     // reference
#include "milo/lowrank.hpp"  // reference
#include "milo/pack.hpp"     // reference
#include "milo/quant.hpp"    // reference
#include "milo_b200.hpp"     // this repo

namespace bind {

milo::b200::PackedInt3Matrix to_b200(const milo::PackedInt3Matrix& p) {
  milo::b200::PackedInt3Matrix q;
  q.rows = p.rows;
  q.cols = p.cols;
  q.layout = p.layout == milo::PackLayout::Linear ? milo::b200::PackLayout::Linear : milo::b200::PackLayout::Tiled16x64;
  q.split = p.split;
  q.mode = p.mode == milo::DequantMode::Symmetric ? milo::b200::DequantMode::Symmetric
                                                 : milo::b200::DequantMode::Asymmetric;
  q.group_size = p.group_size;
  q.words = p.words;
  q.plane_a = p.plane_a;
  q.plane_b = p.plane_b;
  q.scales = p.scales;  // binary16 bits (milo::half_t is std::uint16_t)
  q.zeros = p.zeros;
  return q;
}
milo::b200::WeightMatrix to_b200(const milo::WeightMatrix& a) {
  milo::b200::WeightMatrix b(a.rows, a.cols);
  b.data = a.data;
  return b;
}
milo::b200::GemmConfig to_b200(const milo::GemmConfig& c) {
  milo::b200::GemmConfig g;
  g.tile_shape = c.tile_shape;
  g.group_size = c.group_size;
  g.mode = c.mode == milo::DequantMode::Symmetric ? milo::b200::DequantMode::Symmetric
                                                 : milo::b200::DequantMode::Asymmetric;
  g.pipeline_depth = c.pipeline_depth;
  g.materialize_compensator = c.materialize_compensator;
  return g;
}
milo::b200::Compensator to_b200(const milo::Compensator& c) {
  milo::b200::Compensator d;
  d.rows = c.rows;
  d.cols = c.cols;
  d.rank = c.rank;
  d.storage = c.storage == milo::CompensatorStorage::Real ? milo::b200::CompensatorStorage::Real
                                                          : milo::b200::CompensatorStorage::SymmInt3;
  d.U = c.U;
  d.V = c.V;
  d.qU = {c.qU.rows, c.qU.cols, c.qU.group_size, c.qU.codes, c.qU.scales};
  d.qVt = {c.qVt.rows, c.qVt.cols, c.qVt.group_size, c.qVt.codes, c.qVt.scales};
  return d;
}

}  // namespace bind

// A packed k x n matrix through the reference's public quantize / pack API.
static milo::PackedInt3Matrix make_packed(std::size_t k, std::size_t n, milo::DequantMode mode, uint64_t seed) {
  std::mt19937_64 rng(seed);
  if (mode == milo::DequantMode::Asymmetric) {
    milo::WeightMatrix w(k, n);
    std::normal_distribution<float> dist(0.0f, 0.05f);
    for (float& v : w.data) v = dist(rng);
    milo::QuantConfig qc;
    const milo::QuantParams qp = milo::init_quant_params(w, qc);
    return milo::pack_linear(milo::quantize(w, qp.scales, qp.zeros, qc));
  }
  std::vector<std::uint8_t> codes(k * n);
  std::uniform_int_distribution<int> cd(0, 7);
  for (auto& c : codes) c = static_cast<std::uint8_t>(cd(rng));
  std::vector<float> scales(k * n / 64);
  std::normal_distribution<float> sd(0.0f, 0.05f);
  for (float& s : scales) s = std::fabs(sd(rng)) + 0.01f;
  return milo::pack_linear_symmetric(k, n, codes, scales, 64);
}

static double rel_err(const std::vector<float>& got, const std::vector<float>& want) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < got.size(); ++i) {
    const double d = (double)got[i] - want[i];
    num += d * d;
    den += (double)want[i] * want[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

int main() {
  int fails = 0;
  struct Case {
    std::size_t k, n;
    milo::DequantMode mode;
    std::size_t rank;
  };
  const Case cases[] = {{512, 1024, milo::DequantMode::Asymmetric, 0},
                        {1024, 512, milo::DequantMode::Symmetric, 0},
                        {512, 1024, milo::DequantMode::Asymmetric, 32}};
  for (const Case& c : cases) {
    const milo::PackedInt3Matrix packed = make_packed(c.k, c.n, c.mode, 7 + c.k + c.rank);
    const milo::b200::DeviceWeight dW(bind::to_b200(packed));  // one-time upload + repack
    std::optional<milo::Compensator> comp;
    std::optional<milo::b200::DeviceCompensator> dC;
    if (c.rank > 0) {  // a symm-INT3 factor pair through the reference's own quantizer
      milo::Compensator cc;
      cc.rows = c.k;
      cc.cols = c.n;
      cc.rank = c.rank;
      cc.U.resize(c.k * c.rank);
      cc.V.resize(c.rank * c.n);
      std::mt19937_64 rng(99);
      std::normal_distribution<float> dist(0.0f, 0.05f);
      for (float& v : cc.U) v = dist(rng);
      for (float& v : cc.V) v = dist(rng);
      cc.quantize_symm_int3(64);
      comp = cc;
      dC.emplace(bind::to_b200(cc));
    }
    milo::GemmConfig cfg;
    cfg.mode = c.mode;
    for (std::size_t m : {1u, 7u, 64u}) {
      milo::WeightMatrix A(m, c.k);
      std::mt19937_64 rng(1000 + m);
      std::normal_distribution<float> dist(0.0f, 1.0f);
      for (float& v : A.data) v = dist(rng);
      const milo::WeightMatrix ref = milo::gemm_w3a16(A, packed, comp, cfg);  // reference, CPU
      // was: WeightMatrix C = milo::gemm_w3a16(A, packed, comp, cfg);
      const milo::b200::WeightMatrix C =
          milo::b200::gemm_w3a16(bind::to_b200(A), dW, dC ? &*dC : nullptr, bind::to_b200(cfg));
      const double e = rel_err(C.data, ref.data);
      const bool ok = e <= 1e-5;
      std::printf("%s k=%zu n=%zu mode=%d rank=%zu m=%zu: rel_err %.3g\n", ok ? "ok  " : "FAIL", c.k, c.n,
                  (int)c.mode, c.rank, m, e);
      fails += !ok;
    }
  }
  // the reference's error categories survive the binding: a tile shape the reference
  // rejects (gemm.cpp:23-30) is a b200 ConfigError
  try {
    milo::GemmConfig bad;
    bad.tile_shape = {96, 96};
    const milo::PackedInt3Matrix packed = make_packed(256, 256, milo::DequantMode::Asymmetric, 3);
    const milo::b200::DeviceWeight dW(bind::to_b200(packed));
    milo::WeightMatrix A(1, 256);
    milo::b200::gemm_w3a16(bind::to_b200(A), dW, nullptr, bind::to_b200(bad));
    std::printf("FAIL no ConfigError\n");
    ++fails;
  } catch (const milo::b200::ConfigError&) {
    std::printf("ok   ConfigError for a disallowed tile shape\n");
  }
  std::printf("%s\n", fails ? "binding check FAILED" : "binding check ok");
  return fails ? 1 : 0;
}
