// Run by tests/test_gpu_cpp_api.py on a GPU: the C++ host API (include/milo_b200.hpp)
// end to end -- DeviceWeight / DeviceCompensator from PackedInt3Matrix / Compensator
// values, gemm_w3a16 with host WeightMatrix buffers (the reference's by-value form,
// gemm.hpp:43-48), and a MoELayer forward from host x / router logits.  Inputs are raw
// little-endian files written by the test; the outputs go back the same way and the
// test compares them with the CPU oracle.
//
//   gpu_run <dir>     <dir>/meta.txt:  k n m mode rank   d f E K m2
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "milo_b200.hpp"

using namespace milo::b200;

template <typename T>
static std::vector<T> read_raw(const std::string& path, std::size_t count) {
  std::vector<T> v(count);
  std::ifstream f(path, std::ios::binary);
  if (!f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(count * sizeof(T))))
    throw IoError("cannot read " + path);
  return v;
}
template <typename T>
static void write_raw(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

static PackedInt3Matrix read_packed(const std::string& prefix, std::size_t k, std::size_t n, int mode) {
  PackedInt3Matrix p;
  p.rows = k;
  p.cols = n;
  p.mode = mode == 0 ? DequantMode::Symmetric : DequantMode::Asymmetric;
  p.words = read_raw<std::uint32_t>(prefix + ".words", k * n / 32 * 3);
  p.scales = read_raw<std::uint16_t>(prefix + ".scales", k * n / 64);
  if (mode == 1) p.zeros = read_raw<std::uint16_t>(prefix + ".zeros", k * n / 64);
  return p;
}

int main(int argc, char** argv) {
  if (argc != 2) {
    std::fprintf(stderr, "usage: gpu_run <dir>\n");
    return 2;
  }
  const std::string dir = argv[1];
  std::size_t k, n, m, rank, d, f, E, K, m2;
  int mode;
  {
    std::ifstream meta(dir + "/meta.txt");
    meta >> k >> n >> m >> mode >> rank >> d >> f >> E >> K >> m2;
    if (!meta) {
      std::fprintf(stderr, "bad meta.txt\n");
      return 2;
    }
  }
  try {
    // ---- single linear with a symm-INT3 compensator (configs[0] semantics)
    const DeviceWeight W(read_packed(dir + "/lin", k, n, mode));
    Compensator c;
    c.rows = k;
    c.cols = n;
    c.rank = rank;
    c.storage = CompensatorStorage::SymmInt3;
    const std::size_t gpr = (rank + 63) / 64;
    c.qU.rows = k;
    c.qU.cols = rank;
    c.qU.codes = read_raw<std::uint8_t>(dir + "/lin.qu_codes", k * rank);
    c.qU.scales = read_raw<float>(dir + "/lin.qu_scales", k * gpr);
    c.qVt.rows = n;
    c.qVt.cols = rank;
    c.qVt.codes = read_raw<std::uint8_t>(dir + "/lin.qvt_codes", n * rank);
    c.qVt.scales = read_raw<float>(dir + "/lin.qvt_scales", n * gpr);
    const DeviceCompensator C(c);
    if (C.rank() != rank) throw RankError("compensator rank");
    WeightMatrix A(m, k);
    A.data = read_raw<float>(dir + "/A.f32", m * k);
    GemmConfig cfg;
    cfg.mode = c.rows ? (mode == 0 ? DequantMode::Symmetric : DequantMode::Asymmetric) : cfg.mode;
    const WeightMatrix out = gemm_w3a16(A, W, &C, cfg);
    write_raw(dir + "/C.f32", out.data);

    // ---- MoE layer: E experts (w1, w3: d x f; w2: f x d), top-K, no compensators
    std::vector<DeviceWeight> mats;
    mats.reserve(3 * E);
    for (std::size_t e = 0; e < E; ++e)
      for (int j = 0; j < 3; ++j)
        mats.emplace_back(read_packed(dir + "/e" + std::to_string(e) + "_" + std::to_string(j), j < 2 ? d : f,
                                      j < 2 ? f : d, 1));
    std::vector<ExpertRef> experts;
    for (std::size_t e = 0; e < E; ++e) experts.push_back({&mats[3 * e], &mats[3 * e + 1], &mats[3 * e + 2]});
    const MoELayer layer(experts, {}, static_cast<int>(K));
    WeightMatrix x(m2, d), logits(m2, E);
    x.data = read_raw<float>(dir + "/x.f32", m2 * d);
    logits.data = read_raw<float>(dir + "/logits.f32", m2 * E);
    write_raw(dir + "/moe.f32", layer.forward(x, logits).data);
    // a shape error surfaces as the reference's category
    bool shape_error = false;
    try {
      WeightMatrix bad(m, k + 32);
      gemm_w3a16(bad, W, &C, cfg);
    } catch (const ShapeError&) {
      shape_error = true;
    }
    if (!shape_error) throw MiloError(ErrorCode::Argument, "no ShapeError for A.cols != k");
  } catch (const MiloError& e) {
    std::fprintf(stderr, "MiloError (%d): %s\n", static_cast<int>(e.code()), e.what());
    return 1;
  }
  std::printf("gpu_run ok\n");
  return 0;
}
