// Compiled and run by tests/test_capi.py (CPU): exercises the C++ host API's
// host-side validation through the C ABI (no GPU needed for these paths).
#include <cstdio>
#include "milo_b200.hpp"

using namespace milo::b200;

int main() {
  int fails = 0;
  auto expect = [&](const char* what, auto&& fn, ErrorCode want) {
    try {
      fn();
      std::printf("FAIL %s: no exception\n", what);
      ++fails;
    } catch (const MiloError& e) {
      if (e.code() != want) {
        std::printf("FAIL %s: code %d\n", what, (int)e.code());
        ++fails;
      }
    }
  };
  // container loaders (no device here: only that they compile and report a missing file)
  expect("load missing", [&] { DeviceWeight::load("/nonexistent.milo"); }, ErrorCode::Io);
  expect("comp missing", [&] { DeviceCompensator::load("/nonexistent.u.milo", "/nonexistent.v.milo"); },
         ErrorCode::Io);
  PackedInt3Matrix p;
  p.rows = 16;
  p.cols = 48;  // not a multiple of 32
  expect("cols%32", [&] { DeviceWeight w(p); }, ErrorCode::Shape);
  p.cols = 64;
  p.words.assign(16 * 64 / 32 * 3 - 1, 0u);  // wrong length
  p.scales.assign(16, 0);
  expect("word count", [&] { DeviceWeight w(p); }, ErrorCode::Format);
  p.rows = 0;
  expect("empty", [&] { DeviceWeight w(p); }, ErrorCode::Shape);
  if (milo_abi_version() != MILO_B200_ABI_VERSION) ++fails;
  std::printf("%s\n", fails ? "abi_check FAILED" : "abi_check ok");
  return fails ? 1 : 0;
}
