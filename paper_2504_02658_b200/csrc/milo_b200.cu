// C-ABI implementation (include/milo_b200.h): handle management, reference-
// order validation, workspace planning and kernel launches.  Host C++.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <chrono>
#include <functional>
#include <map>
#include <atomic>
#include <climits>
#include <mutex>
#include <string>
#include <utility>
#include <vector>
#include <type_traits>

#include <cuda_fp16.h>

#include "../../include/milo_b200.h"
#include "gemv.cuh"
#include "kernels.cuh"
#include "lorc.cuh"
#include "moe.cuh"
#include "decode.cuh"
#include "hdec.cuh"
#include "prefill.cuh"

using namespace milo_dev;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;

milo_status fail(milo_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e__ = (expr);                                                            \
    if (e__ != cudaSuccess)                                                              \
      return fail(MILO_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e__));      \
  } while (0)

struct DeviceProps {
  int sms = 0;
  int major = 0;
  bool ok = false;
};

DeviceProps device_props() {
  static std::mutex mu;
  static DeviceProps cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return {};
  std::lock_guard<std::mutex> lock(mu);
  DeviceProps& p = cache[dev];
  if (!p.ok) {
    cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&p.major, cudaDevAttrComputeCapabilityMajor, dev);
    p.ok = p.sms > 0;
    // Per-call workspaces come from the stream-ordered pool; keep freed
    // blocks cached instead of returning them to the driver at every sync.
    cudaMemPool_t pool;
    if (p.ok && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t threshold = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
  }
  return p;
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
// Same, and the smallest shared-memory carveout that holds it: the rest of the
// SM's 256 KB unified L1 / shared storage stays L1 (the decode kernel's
// activation rows are read through L1).
template <typename K>
cudaError_t set_smem_min_carveout(K kernel, int bytes) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  const int pct = (int)(((int64_t)bytes + 2048) * 100 / (228 * 1024)) + 1;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
}

// Host -> device uploads of per-call tables go through a per-thread pinned
// staging buffer: a cudaMemcpyAsync from pageable memory is a synchronous staged
// copy (~5-10 us each; a MoE prefill call issues ~10 of them while the GPU idles).
// pin_begin() at the start of a launch sequence waits for the previous sequence's
// copies (event), pin_end() records that event.
struct PinStage {
  uint8_t* base = nullptr;
  size_t cap = 0, off = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
  // Two-pass sequences (moe_prefill): mode 1 records the uploads of a dry run
  // (no launches) at stage offsets mirroring their device offsets, pin_flush()
  // issues them as few coalesced copies, mode 2 replays the sequence with the
  // uploads already in flight, so no copy sits between two kernels.
  int mode = 0;
  struct Rec { uint8_t* dst; size_t off, bytes; };
  std::vector<Rec> rec;
  uint8_t *lo = nullptr, *hi = nullptr;  // device range in which recorded copies may be merged
};
thread_local PinStage g_pin;
thread_local bool g_dry = false;  // dry run: launch() and ProfScope do nothing
void pin_begin() {
  if (g_pin.pending) {
    cudaEventSynchronize(g_pin.ev);
    g_pin.pending = false;
  }
  g_pin.off = 0;
}
void pin_end(cudaStream_t s) {
  if (!g_pin.ev) cudaEventCreateWithFlags(&g_pin.ev, cudaEventDisableTiming);
  cudaEventRecord(g_pin.ev, s);
  g_pin.pending = true;
}
cudaError_t pin_reserve(size_t need, cudaStream_t s) {  // grow, keeping this sequence's staged bytes
  if (need <= g_pin.cap) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(s);  // nothing of this sequence may still read the old buffer
  if (e != cudaSuccess) return e;
  const size_t cap = std::max<size_t>({need, 2 * g_pin.cap, (size_t)1 << 20});
  uint8_t* nb = nullptr;
  e = cudaMallocHost(&nb, cap);
  if (e != cudaSuccess) return e;
  if (g_pin.base) {
    std::memcpy(nb, g_pin.base, g_pin.off);
    cudaFreeHost(g_pin.base);
  }
  g_pin.base = nb;
  g_pin.cap = cap;
  return cudaSuccess;
}
cudaError_t h2d_async(void* dst_, const void* src, size_t bytes, cudaStream_t s) {
  if (!bytes || !src || g_pin.mode == 2) return cudaSuccess;
  uint8_t* dst = static_cast<uint8_t*>(dst_);
  size_t off = g_pin.off;
  if (g_pin.mode == 1 && !g_pin.rec.empty()) {  // mirror the device layout inside the merge range
    const PinStage::Rec& l = g_pin.rec.back();
    if (dst >= l.dst + l.bytes && dst >= g_pin.lo && dst + bytes <= g_pin.hi && l.dst >= g_pin.lo &&
        dst - l.dst < (1 << 16))
      off = std::max(off, l.off + (size_t)(dst - l.dst));
  }
  cudaError_t e = pin_reserve(off + bytes, s);
  if (e != cudaSuccess) return g_pin.mode == 1 ? e : cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  std::memcpy(g_pin.base + off, src, bytes);
  g_pin.off = (off + bytes + 255) & ~size_t(255);
  if (g_pin.mode == 1) {
    g_pin.rec.push_back({dst, off, bytes});
    return cudaSuccess;
  }
  return cudaMemcpyAsync(dst, g_pin.base + off, bytes, cudaMemcpyHostToDevice, s);
}
// Issues the recorded uploads: runs whose device and stage offsets advance
// together inside the merge range become one copy (the gaps are unused table
// padding).
cudaError_t pin_flush(cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  size_t i = 0;
  while (i < g_pin.rec.size() && e == cudaSuccess) {
    const PinStage::Rec& a = g_pin.rec[i];
    size_t end = a.bytes, j = i + 1;
    for (; j < g_pin.rec.size(); ++j) {
      const PinStage::Rec& b = g_pin.rec[j];
      if (!(a.dst >= g_pin.lo && b.dst + b.bytes <= g_pin.hi && b.dst >= a.dst + end &&
            (size_t)(b.dst - a.dst) == b.off - a.off))
        break;
      end = (size_t)(b.dst - a.dst) + b.bytes;
    }
    e = cudaMemcpyAsync(a.dst, g_pin.base + a.off, end, cudaMemcpyHostToDevice, s);
    i = j;
  }
  g_pin.rec.clear();
  return e;
}

// Launch with programmatic dependent launch allowed (the kernel itself calls
// griddepcontrol.wait before touching the previous grid's outputs).
template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t stream, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (g_dry) return cudaSuccess;
  ++g_launches;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Optional per-kernel CUDA-event timing (milo_profile_*), recorded on the
// launching stream around selected launches.  Off by default.
enum ProfKind { kProfGemv1 = 0, kProfGemv2 = 1, kProfLorc = 2, kProfOther = 3, kProfKinds = 4 };
struct ProfState {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kProfKinds];
};
thread_local ProfState g_prof;

struct ProfScope {
  cudaEvent_t b = nullptr, e = nullptr;
  cudaStream_t s;
  int kind;
  ProfScope(int k, cudaStream_t st) : s(st), kind(k) {
    if (!g_prof.on || g_dry) return;
    cudaEventCreate(&b);
    cudaEventCreate(&e);
    cudaEventRecord(b, s);
  }
  ~ProfScope() {
    if (!b) return;
    cudaEventRecord(e, s);
    g_prof.ev[kind].push_back({b, e});
  }
};

// Bump allocator over one stream-ordered allocation.
struct Arena {
  size_t size = 0;
  size_t take(size_t bytes) {
    size_t off = (size + 255) & ~size_t(255);
    size = off + bytes;
    return off;
  }
};

// MILO_LEGACY=1 selects the multi-launch decode path (A/B comparisons only).
bool legacy_path() {
  static const bool v = [] {
    const char* e = getenv("MILO_LEGACY");
    return e != nullptr && e[0] == '1';
  }();
  return v;
}

bool tile_allowed(int tk, int tn) {
  return (tk == 64 && tn == 256) || (tk == 128 && tn == 128) || (tk == 256 && tn == 64);
}

}  // namespace

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
struct milo_weight {
  uint64_t rows = 0, cols = 0;
  int32_t mode = 1;
  uint64_t group_size = 64;
  bool has_zeros = false;
  uint8_t* tiles = nullptr;  // macro-tile layout (null when the layout is not representable)
  uint64_t bytes = 0;
};

struct milo_comp {
  uint64_t rows = 0, cols = 0, rank = 0;
  int32_t storage = 1;
  uint64_t group_size = 64;
  void* mem = nullptr;
  uint8_t* ucodes = nullptr;  // k x rank
  float* uscales = nullptr;   // k x gpr
  uint8_t* vcodes = nullptr;  // n x rank (qVt)
  float* vscales = nullptr;   // n x gpr
  float* ureal = nullptr;     // k x rank
  float* vreal = nullptr;     // n x rank (V^T)
  int32_t gpr = 0;
  // decode-kernel layouts (decode.cuh): U pseudo tiles, V^T fragment tiles, V steps
  void* dmem = nullptr;
  uint8_t* upt = nullptr;
  uint8_t* vft = nullptr;
  float* vstep = nullptr;
  int32_t r16 = 0;
  // prefill (tcgen05) layout: V^T operand images [n/128][r/64][hi, lo][16 KB]
  void* pmem = nullptr;
  uint8_t* vimg = nullptr;
  int32_t rch = 0;
};

// ---------------------------------------------------------------------------
// Compensator layouts of the decode kernel (decode.cuh), built on the host once
// per compensator.  U pseudo tiles: A operand of t = x U (rows = 16 rank
// columns, cols = 32 k); V fragment tiles: A operand of t V (rows = 64 n of a
// slab, cols = 16 ranks per step).  int3: exact codes (pad code 4 == 0.0) and
// fp32 steps s * (2/7) (lowrank.cpp:122-134, the same fp32 expression);
// real: binary16 hi + lo split of the fp32 factors (pad 0).
// ---------------------------------------------------------------------------
namespace {

// binary32 -> binary16, round to nearest even (branch-free; NaN stays NaN):
// the host-side half(A) of the reference's activations (half.hpp float_to_half).
inline uint16_t f32_to_f16_rne(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  x &= 0x7FFFFFFFu;
  uint16_t o;
  if (x >= 0x47800000u) {  // overflow -> inf, NaN -> quiet NaN
    o = x > 0x7F800000u ? 0x7E00u : 0x7C00u;
  } else if (x < 0x38800000u) {  // subnormal / zero: add the magic 0.5, let the FPU round
    float t;
    std::memcpy(&t, &x, 4);
    t += 0.5f;
    uint32_t ti;
    std::memcpy(&ti, &t, 4);
    o = (uint16_t)(ti - 0x3F000000u);
  } else {
    const uint32_t mant_odd = (x >> 13) & 1u;
    x += 0xC8000FFFu + mant_odd;  // rebias exponent (15 - 127) << 23 and round
    o = (uint16_t)(x >> 13);
  }
  return (uint16_t)(o | sign);
}

uint16_t h16(float f) {
  const __half h = __float2half_rn(f);
  return *reinterpret_cast<const uint16_t*>(&h);
}
float f16f(uint16_t b) {
  __half h;
  *reinterpret_cast<uint16_t*>(&h) = b;
  return __half2float(h);
}

cudaError_t build_decode_layouts(milo_comp* c, const milo_comp_desc* d) {
  const uint64_t k = d->rows, n = d->cols, r = d->rank;
  const bool real = d->storage != 1;
  const uint64_t r16 = (r + 15) / 16 * 16, nks = r16 / 16, gpr = (r + 63) / 64;
  c->r16 = (int32_t)r16;
  if (k % 32 != 0 || n % 64 != 0) return cudaSuccess;  // not a GEMM shape: no decode layout
  const uint64_t upt_b = nks * (k / 32) * (real ? kPseudoRealBytes : kPseudoInt3Bytes);
  const uint64_t vft_b = (n / 64) * nks * (real ? kVftRealBytes : kVftInt3Bytes);
  const uint64_t vst_b = real ? 0 : n * gpr * 4;
  std::vector<uint8_t> host(upt_b + vft_b + vst_b, 0);
  uint8_t* upt = host.data();
  uint8_t* vft = upt + upt_b;
  float* vst = reinterpret_cast<float*>(vft + vft_b);
  auto ucode = [&](uint64_t kk, uint64_t j) -> uint8_t { return j < r ? d->qu_codes[kk * r + j] : 4; };
  auto vcode = [&](uint64_t nn, uint64_t j) -> uint8_t { return j < r ? d->qvt_codes[nn * r + j] : 4; };
  auto uval = [&](uint64_t kk, uint64_t j) -> float { return j < r ? d->U[kk * r + j] : 0.0f; };
  auto vval = [&](uint64_t nn, uint64_t j) -> float { return j < r ? d->V[j * n + nn] : 0.0f; };
  auto put_split = [](uint8_t* dst, float v) {  // hi at dst, lo at dst + 16
    const uint16_t hi = h16(v);
    const uint16_t lo = h16(v - f16f(hi));
    memcpy(dst, &hi, 2);
    memcpy(dst + 16, &lo, 2);
  };
  for (uint64_t rc = 0; rc < nks; ++rc)
    for (uint64_t kt = 0; kt < k / 32; ++kt) {
      uint8_t* tile = upt + (rc * (k / 32) + kt) * (real ? kPseudoRealBytes : kPseudoInt3Bytes);
      for (int lane = 0; lane < 32; ++lane)
        for (int ks = 0; ks < 2; ++ks)
          for (int a = 0; a < 4; ++a)
            for (int h = 0; h < 2; ++h) {
              const int g = lane >> 2, q = lane & 3;
              const uint64_t j = rc * 16 + g + 8 * (a & 1);
              const uint64_t kk = kt * 32 + 16 * ks + 2 * q + 8 * (a >> 1) + h;
              if (!real)
                tile[lane * 16 + ks * 8 + 2 * a + h] = ucode(kk, j);
              else
                put_split(tile + lane * 64 + ks * 32 + a * 4 + h * 2, uval(kk, j));
            }
      if (!real) {
        float* st = reinterpret_cast<float*>(tile + 512);
        const uint64_t grp = (rc * 16) / 64;
        for (int i = 0; i < 32; ++i) st[i] = d->qu_scales[(kt * 32 + i) * gpr + grp] * (2.0f / 7.0f);
      }
    }
  for (uint64_t slab = 0; slab < n / 64; ++slab)
    for (uint64_t ks = 0; ks < nks; ++ks) {
      uint8_t* tile = vft + (slab * nks + ks) * (real ? kVftRealBytes : kVftInt3Bytes);
      for (int lane = 0; lane < 32; ++lane)
        for (int i = 0; i < 4; ++i)
          for (int a = 0; a < 4; ++a)
            for (int h = 0; h < 2; ++h) {
              const int g = lane >> 2, q = lane & 3;
              const uint64_t nn = slab * 64 + 16 * i + g + 8 * (a & 1);
              const uint64_t j = 16 * ks + 2 * q + 8 * (a >> 1) + h;
              if (!real)
                tile[lane * 32 + i * 8 + 2 * a + h] = vcode(nn, j);
              else
                put_split(tile + lane * 128 + i * 32 + a * 4 + h * 2, vval(nn, j));
            }
    }
  if (!real)
    for (uint64_t nn = 0; nn < n; ++nn)
      for (uint64_t gg = 0; gg < gpr; ++gg) vst[nn * gpr + gg] = d->qvt_scales[nn * gpr + gg] * (2.0f / 7.0f);
  cudaError_t e = cudaMalloc(&c->dmem, host.size());
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(c->dmem, host.data(), host.size(), cudaMemcpyHostToDevice);
  c->upt = static_cast<uint8_t*>(c->dmem);
  c->vft = c->upt + upt_b;
  c->vstep = real ? nullptr : reinterpret_cast<float*>(c->vft + vft_b);
  if (e != cudaSuccess || n % kPfM != 0) return e;
  // prefill V^T images: row = output column n of the 128-tile, K = rank (64 per
  // chunk), SW128 K-major binary16, value v = step * (c - 4) (lowrank.cpp:122-134)
  // or real V, split into hi + lo halves
  const uint64_t rch = (r + 63) / 64;
  c->rch = (int32_t)rch;
  std::vector<uint8_t> img((n / kPfM) * rch * 2 * kPfImg, 0);
  for (uint64_t nn = 0; nn < n; ++nn)
    for (uint64_t j = 0; j < rch * 64; ++j) {
      float v = 0.0f;
      if (j < r) {
        if (!real)
          v = (d->qvt_scales[nn * gpr + j / 64] * (2.0f / 7.0f)) * ((float)d->qvt_codes[nn * r + j] - 4.0f);
        else
          v = d->V[j * n + nn];
      }
      const uint16_t hi = h16(v), lo = h16(v - f16f(hi));
      const uint64_t tile = nn / kPfM, row = nn % kPfM, ch = j / 64, jj = j % 64;
      const uint64_t off = row * 128 + (((jj >> 3) ^ (row & 7)) << 4) + (jj & 7) * 2;
      uint8_t* b = img.data() + ((tile * rch + ch) * 2) * kPfImg;
      memcpy(b + off, &hi, 2);
      memcpy(b + kPfImg + off, &lo, 2);
    }
  e = cudaMalloc(&c->pmem, img.size());
  if (e == cudaSuccess) e = cudaMemcpy(c->pmem, img.data(), img.size(), cudaMemcpyHostToDevice);
  c->vimg = static_cast<uint8_t*>(c->pmem);
  return e;
}

}  // namespace

extern "C" {

const char* milo_last_error(void) { return g_err.c_str(); }
int milo_abi_version(void) { return MILO_B200_ABI_VERSION; }
uint64_t milo_launch_count(void) { return g_launches; }

const char* milo_status_name(milo_status s) {
  switch (s) {
    case MILO_OK: return "ok";
    case MILO_ERR_FORMAT: return "format";
    case MILO_ERR_DATA: return "data";
    case MILO_ERR_IO: return "io";
    case MILO_ERR_SHAPE: return "shape";
    case MILO_ERR_RANK: return "rank";
    case MILO_ERR_NUMERIC: return "numeric";
    case MILO_ERR_STAT: return "stat";
    case MILO_ERR_PLAN: return "plan";
    case MILO_ERR_RANGE: return "range";
    case MILO_ERR_CONFIG: return "config";
    case MILO_ERR_CUDA: return "cuda";
    case MILO_ERR_ARGUMENT: return "argument";
  }
  return "unknown";
}

void milo_profile_enable(int32_t on) { g_prof.on = on != 0; }

// Sums the recorded durations of one kernel kind (synchronizing on the last
// event), returns the count, and releases the events.
int64_t milo_profile_read(int32_t kind, double* total_ms) {
  if (kind < 0 || kind >= kProfKinds) return -1;
  double tot = 0.0;
  auto& v = g_prof.ev[kind];
  for (auto& pe : v) {
    float ms = 0.0f;
    cudaEventSynchronize(pe.second);
    cudaEventElapsedTime(&ms, pe.first, pe.second);
    tot += ms;
    cudaEventDestroy(pe.first);
    cudaEventDestroy(pe.second);
  }
  const int64_t n = (int64_t)v.size();
  v.clear();
  if (total_ms) *total_ms = tot;
  return n;
}

milo_status milo_device_check(void) {
  DeviceProps p = device_props();
  if (!p.ok) return fail(MILO_ERR_CUDA, "no CUDA device");
  if (p.major != 10) return fail(MILO_ERR_CUDA, "device is sm_%d0, this library is sm_100a only", p.major);
  cudaFuncAttributes fa;
  CUDA_TRY(cudaFuncGetAttributes(&fa, gemv_w3a16_kernel<2, 1>));
  CUDA_TRY(cudaFuncGetAttributes(&fa, lorc_t_kernel));
  return MILO_OK;
}

milo_status milo_weight_create(const milo_packed_desc* d, milo_weight** out) {
  if (!d || !out) return fail(MILO_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  // PackedInt3Matrix invariants (pack.cpp:72-76, pack.hpp:47-58).
  if (d->rows == 0 || d->cols == 0) return fail(MILO_ERR_SHAPE, "cannot pack an empty matrix");
  if (d->cols % 32 != 0) return fail(MILO_ERR_SHAPE, "cols %llu not a multiple of 32", (unsigned long long)d->cols);
  if (d->group_size == 0 || (d->rows * d->cols) % d->group_size != 0)
    return fail(MILO_ERR_SHAPE, "group_size does not divide rows*cols");
  if (d->layout != 0 && d->layout != 1) return fail(MILO_ERR_FORMAT, "unknown layout %d", d->layout);
  if (d->mode != 0 && d->mode != 1) return fail(MILO_ERR_FORMAT, "unknown mode %d", d->mode);
  if (d->layout == 1 && (d->rows % 16 != 0 || d->cols % 64 != 0))
    return fail(MILO_ERR_SHAPE, "tiled layout needs rows %% 16 == 0 and cols %% 64 == 0");
  const uint64_t groups = d->rows * d->cols / 32;
  const uint64_t qg = d->rows * d->cols / d->group_size;
  if (d->split) {
    if (!d->plane_a || !d->plane_b || d->n_plane_a != groups * 2 || d->n_plane_b != groups)
      return fail(MILO_ERR_FORMAT, "split planes must hold %llu + %llu words",
                  (unsigned long long)(groups * 2), (unsigned long long)groups);
  } else if (!d->words || d->n_words != groups * 3) {
    return fail(MILO_ERR_FORMAT, "words must hold %llu words", (unsigned long long)(groups * 3));
  }
  if (!d->scales || d->n_scales != qg) return fail(MILO_ERR_FORMAT, "scales must hold %llu values", (unsigned long long)qg);
  if (d->zeros && d->n_zeros != qg && d->n_zeros != 0)
    return fail(MILO_ERR_FORMAT, "zeros must hold %llu values or be empty", (unsigned long long)qg);
  DeviceProps props = device_props();
  if (!props.ok) return fail(MILO_ERR_CUDA, "no CUDA device");

  auto* w = new milo_weight();
  w->rows = d->rows;
  w->cols = d->cols;
  w->mode = d->mode;
  w->group_size = d->group_size;
  w->has_zeros = d->zeros != nullptr && d->n_zeros == qg;
  const bool representable = d->group_size == 64 && d->rows % 32 == 0 && d->cols % 64 == 0 &&
                             (d->mode == 0 || w->has_zeros);
  if (!representable) {  // gemm_w3a16 rejects these inputs (gemm.cpp:121-134)
    *out = w;
    return MILO_OK;
  }
  w->bytes = d->rows * d->cols / 2048 * kTileBytes;
  const size_t word_bytes = groups * 3 * 4, meta_bytes = qg * 2;
  void* staging = nullptr;
  cudaError_t e = cudaMalloc(&w->tiles, w->bytes);
  if (e == cudaSuccess) e = cudaMalloc(&staging, word_bytes + 2 * meta_bytes + 64);
  if (e != cudaSuccess) {
    cudaFree(w->tiles);
    delete w;
    return fail(MILO_ERR_CUDA, "cudaMalloc failed: %s", cudaGetErrorString(e));
  }
  uint8_t* st = static_cast<uint8_t*>(staging);
  uint32_t* dwords = reinterpret_cast<uint32_t*>(st);
  uint16_t* dscales = reinterpret_cast<uint16_t*>(st + word_bytes);
  uint16_t* dzeros = reinterpret_cast<uint16_t*>(st + word_bytes + meta_bytes);
  RefStream rs{};
  rs.rows = d->rows;
  rs.cols = d->cols;
  rs.layout = d->layout;
  rs.split = d->split;
  if (d->split) {
    e = cudaMemcpy(dwords, d->plane_a, groups * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dwords + groups * 2, d->plane_b, groups * 4, cudaMemcpyHostToDevice);
    rs.plane_a = dwords;
    rs.plane_b = dwords + groups * 2;
  } else {
    e = cudaMemcpy(dwords, d->words, word_bytes, cudaMemcpyHostToDevice);
    rs.words = dwords;
  }
  if (e == cudaSuccess) e = cudaMemcpy(dscales, d->scales, meta_bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && w->has_zeros) e = cudaMemcpy(dzeros, d->zeros, meta_bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const uint64_t threads = (d->rows * d->cols / 2048) * 32;
    ++g_launches;
    repack_codes_kernel<<<(unsigned)((threads + 255) / 256), 256>>>(rs, w->tiles, d->rows, d->cols);
    const uint64_t mthreads = d->rows * (d->cols / 64);
    ++g_launches;
    repack_meta_kernel<<<(unsigned)((mthreads + 255) / 256), 256>>>(dscales, dzeros, d->mode, w->tiles,
                                                                   d->rows, d->cols);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(staging);
  if (e != cudaSuccess) {
    cudaFree(w->tiles);
    delete w;
    return fail(MILO_ERR_CUDA, "repack failed: %s", cudaGetErrorString(e));
  }
  *out = w;
  return MILO_OK;
}

milo_status milo_weight_destroy(milo_weight* w) {
  if (!w) return MILO_OK;
  if (w->tiles) cudaFree(w->tiles);
  delete w;
  return MILO_OK;
}

milo_status milo_weight_info(const milo_weight* w, uint64_t* rows, uint64_t* cols, int32_t* mode,
                             uint64_t* device_bytes) {
  if (!w) return fail(MILO_ERR_ARGUMENT, "null weight");
  if (rows) *rows = w->rows;
  if (cols) *cols = w->cols;
  if (mode) *mode = w->mode;
  if (device_bytes) *device_bytes = w->bytes;
  return MILO_OK;
}

milo_status milo_comp_info(const milo_comp* c, uint64_t* rows, uint64_t* cols, uint64_t* rank,
                           int32_t* storage) {
  if (!c) return fail(MILO_ERR_ARGUMENT, "null compensator");
  if (rows) *rows = c->rows;
  if (cols) *cols = c->cols;
  if (rank) *rank = c->rank;
  if (storage) *storage = c->storage;
  return MILO_OK;
}

static milo_status unpack_common(const milo_weight* w, int what, int mode, void* out, void* stream) {
  if (!w || !out) return fail(MILO_ERR_ARGUMENT, "null argument");
  if (what == 1 && mode == 1 && !w->has_zeros)
    return fail(MILO_ERR_CONFIG, "asymmetric de-quantization needs zero-points");
  if (!w->tiles)
    return fail(MILO_ERR_CONFIG, "device layout needs group_size 64, rows %% 32 == 0, cols %% 64 == 0");
  if (what == 1 && mode != w->mode)
    return fail(MILO_ERR_CONFIG, "device de-quantization uses the weight's own mode");
  const uint64_t threads = (w->rows * w->cols / 2048) * 32;
  ++g_launches;
  unpack_tiles_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      w->tiles, w->rows, w->cols, w->mode, what, out);
  CUDA_TRY(cudaGetLastError());
  return MILO_OK;
}

milo_status milo_unpack_codes(const milo_weight* w, uint8_t* out, void* stream) {
  return unpack_common(w, 0, w ? w->mode : 0, out, stream);
}

milo_status milo_dequant_half(const milo_weight* w, int32_t mode, uint16_t* out, void* stream) {
  return unpack_common(w, 1, mode, out, stream);
}

milo_status milo_comp_create(const milo_comp_desc* d, milo_comp** out) {
  if (!d || !out) return fail(MILO_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  auto* c = new milo_comp();
  c->rows = d->rows;
  c->cols = d->cols;
  c->rank = d->rank;
  c->storage = d->storage;
  c->group_size = d->group_size;
  if (d->rank == 0) {
    *out = c;
    return MILO_OK;
  }
  if (d->storage == 1 && d->group_size != 64) {
    delete c;
    return fail(MILO_ERR_CONFIG, "device compensator needs symm-int3 group_size 64");
  }
  const uint64_t k = d->rows, n = d->cols, r = d->rank;
  c->gpr = (int32_t)((r + 63) / 64);
  Arena ar;
  size_t o_uc = 0, o_us = 0, o_vc = 0, o_vs = 0, o_ur = 0, o_vr = 0;
  if (d->storage == 1) {
    if (!d->qu_codes || !d->qu_scales || !d->qvt_codes || !d->qvt_scales) {
      delete c;
      return fail(MILO_ERR_ARGUMENT, "symm-int3 compensator arrays missing");
    }
    o_uc = ar.take(k * r);
    o_us = ar.take(k * c->gpr * 4);
    o_vc = ar.take(n * r);
    o_vs = ar.take(n * c->gpr * 4);
  } else {
    if (!d->U || !d->V) {
      delete c;
      return fail(MILO_ERR_ARGUMENT, "real compensator factors missing");
    }
    o_ur = ar.take(k * r * 4);
    o_vr = ar.take(n * r * 4);
  }
  cudaError_t e = cudaMalloc(&c->mem, ar.size);
  if (e != cudaSuccess) {
    delete c;
    return fail(MILO_ERR_CUDA, "cudaMalloc failed: %s", cudaGetErrorString(e));
  }
  uint8_t* base = static_cast<uint8_t*>(c->mem);
  if (d->storage == 1) {
    c->ucodes = base + o_uc;
    c->uscales = reinterpret_cast<float*>(base + o_us);
    c->vcodes = base + o_vc;
    c->vscales = reinterpret_cast<float*>(base + o_vs);
    e = cudaMemcpy(c->ucodes, d->qu_codes, k * r, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(c->uscales, d->qu_scales, k * c->gpr * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(c->vcodes, d->qvt_codes, n * r, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(c->vscales, d->qvt_scales, n * c->gpr * 4, cudaMemcpyHostToDevice);
  } else {
    c->ureal = reinterpret_cast<float*>(base + o_ur);
    c->vreal = reinterpret_cast<float*>(base + o_vr);
    std::vector<float> vt(n * r);
    for (uint64_t j = 0; j < n; ++j)
      for (uint64_t q = 0; q < r; ++q) vt[j * r + q] = d->V[q * n + j];
    e = cudaMemcpy(c->ureal, d->U, k * r * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(c->vreal, vt.data(), n * r * 4, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = build_decode_layouts(c, d);
  if (e != cudaSuccess) {
    cudaFree(c->mem);
    if (c->dmem) cudaFree(c->dmem);
    delete c;
    return fail(MILO_ERR_CUDA, "upload failed: %s", cudaGetErrorString(e));
  }
  *out = c;
  return MILO_OK;
}

milo_status milo_comp_destroy(milo_comp* c) {
  if (!c) return MILO_OK;
  if (c->mem) cudaFree(c->mem);
  if (c->dmem) cudaFree(c->dmem);
  if (c->pmem) cudaFree(c->pmem);
  delete c;
  return MILO_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// GEMM
// ---------------------------------------------------------------------------
namespace {

void fill_comp(GemvProblem& p, int mat, const milo_comp* c) {
  if (!c || c->rank == 0) return;
  p.rank[mat] = (int32_t)c->rank;
  p.vgpr[mat] = c->gpr;
  p.vcodes[mat] = c->vcodes;
  p.vscales[mat] = c->vscales;
  p.vreal[mat] = c->vreal;
  p.ucodes[mat] = c->ucodes;
  p.uscales[mat] = c->uscales;
  p.ureal[mat] = c->ureal;
}

// Workspace of one grouped GEMM launch (sizes in bytes).
template <int NT, int NMAT>
struct GroupedWs {
  using CF = GemvCfg<NT, NMAT>;
  static size_t ws_bytes(int sms) { return (size_t)sms * CF::kWarps * 2 * CF::kPartFloats * 4; }
  static size_t full_bytes(int64_t slabs) { return (size_t)slabs * CF::kPartFloats * 4; }
  // worst case chunk count: real (f32) U rows at the largest rank
  static int lorc_chunks(int64_t k, int rank) {
    return (int)((k + lorc_rows(std::max(rank, 1), 4) - 1) / lorc_rows(std::max(rank, 1), 4));
  }
  static size_t lorc_bytes(int64_t problems, int64_t k, int rank) {
    return (size_t)problems * 2 * lorc_chunks(k, rank) * CF::kMPad * std::max(rank, 1) * 4;
  }
};

// t = A U (lorc_t_kernel, when any rank > 0) -> GEMM with in-kernel fix-up and
// epilogue (+ t V, SwiGLU / store).  Both PDL-chained on `stream`.
template <int NT, int NMAT>
milo_status run_grouped(const GemvProblem* problems, const int32_t* n_problems,
                        int64_t problems_max, int64_t slabs_max, int64_t k_max, int rank_max,
                        float* ws, float* full,
                        int32_t* slab_counters, float* lorc_partial, int32_t* lorc_counters,
                        cudaStream_t stream, int sms, int prof_kind) {
  using CF = GemvCfg<NT, NMAT>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    CUDA_TRY(set_smem(gemv_w3a16_kernel<NT, NMAT>, CF::kBytes));
    CUDA_TRY(set_smem(lorc_t_kernel, kLorcDynSmem));
    configured_dev = dev;
  }
  if (rank_max > 0) {
    LorcArgs la{};
    la.problems = problems;
    la.n_problems = n_problems;
    la.partial = lorc_partial;
    la.counters = lorc_counters;
    la.m_pad = CF::kMPad;
    la.chunks_max = GroupedWs<NT, NMAT>::lorc_chunks(k_max, rank_max);
    la.rank_max = rank_max;
    ProfScope ps(kProfLorc, stream);
    CUDA_TRY(launch(lorc_t_kernel, dim3((unsigned)(problems_max * 2), la.chunks_max),
                    dim3(kLorcThreads), kLorcDynSmem, stream, true, la));
  }
  GemvArgs ga{};
  ga.problems = problems;
  ga.n_problems = n_problems;
  ga.ws = ws;
  ga.full = full;
  ga.counters = slab_counters;
  ga.gw = sms * CF::kWarps;
  {
    ProfScope ps(prof_kind, stream);
    CUDA_TRY(launch(gemv_w3a16_kernel<NT, NMAT>, dim3(sms), dim3(32 * CF::kWarps), CF::kBytes,
                    stream, true, ga));
  }
  ProfScope ps(kProfOther, stream);
  CUDA_TRY(launch(gemv_epilogue_kernel<NT, NMAT>,
                  dim3((unsigned)((slabs_max + kEpiWarps - 1) / kEpiWarps)), dim3(32 * kEpiWarps),
                  0, stream, true, ga));
  return MILO_OK;
}

milo_status validate_gemm(const milo_weight* w, const milo_comp* comp, const milo_gemm_config* cfg,
                          int64_t a_cols) {
  // GemmConfig::validate (gemm.cpp:23-30) then gemm.cpp:120-139, in order.
  if (!tile_allowed(cfg->tile_k, cfg->tile_n))
    return fail(MILO_ERR_CONFIG, "tile shape (%d, %d) not in {(64,256),(128,128),(256,64)}",
                cfg->tile_k, cfg->tile_n);
  if (cfg->group_size != 64) return fail(MILO_ERR_CONFIG, "group size must be 64");
  if (cfg->pipeline_depth < 1) return fail(MILO_ERR_CONFIG, "pipeline depth must be >= 1");
  if (w->group_size != 64) return fail(MILO_ERR_CONFIG, "packed weight group size must be 64");
  if (cfg->mode != w->mode) return fail(MILO_ERR_CONFIG, "config mode does not match the packed weight's mode");
  if (cfg->mode == 1 && !w->has_zeros) return fail(MILO_ERR_CONFIG, "asymmetric mode needs zero-points");
  if (w->rows % (uint64_t)cfg->tile_k != 0 || w->cols % (uint64_t)cfg->tile_n != 0)
    return fail(MILO_ERR_SHAPE, "(k, n) = (%llu, %llu) not a multiple of tile shape (%d, %d)",
                (unsigned long long)w->rows, (unsigned long long)w->cols, cfg->tile_k, cfg->tile_n);
  if ((uint64_t)a_cols != w->rows)
    return fail(MILO_ERR_SHAPE, "A has %lld cols, expected k = %llu", (long long)a_cols,
                (unsigned long long)w->rows);
  if (comp && (comp->rows != w->rows || comp->cols != w->cols))
    return fail(MILO_ERR_SHAPE, "compensator shape does not match the weight");
  if (!w->tiles) return fail(MILO_ERR_CONFIG, "weight has no device layout");
  return MILO_OK;
}

}  // namespace


// ---------------------------------------------------------------------------
// Decode kernel (decode.cuh): per-(device, stream) workspace and launcher.
// ---------------------------------------------------------------------------
namespace {

DecMat make_decmat(const milo_weight* w, const milo_comp* c) {
  DecMat M{};
  M.w = w->tiles;
  M.k = (int32_t)w->rows;
  M.n = (int32_t)w->cols;
  M.mode = w->mode;
  if (c && c->rank > 0 && c->upt) {
    M.upt = c->upt;
    M.vft = c->vft;
    M.vstep = c->vstep;
    M.rank = (int32_t)c->rank;
    M.r16 = c->r16;
    M.gpr = c->gpr;
    M.real = c->storage != 1;
  }
  return M;
}

constexpr int kCntCap = 1 << 17;   // slab counters per phase
constexpr int kCCntCap = 4096;     // d-slab (combine) counters
// control block (int32, zeroed once; counters return to zero after every call,
// flags hold the epoch of the call that set them)
constexpr int kHflagCap = 1 << 17;  // per (block, 64-column slab of h) ready flags
constexpr size_t kCtrlInts = 2 * (size_t)kCntCap + kDecMaxBlocks * 3 + kDecMaxBlocks + kCCntCap +
                             kDecMaxBlocks * 3 + kDecMaxBlocks + kHflagCap;

struct DecodeWs {
  int32_t* ctrl = nullptr;
  int32_t* hctrl = nullptr;  // hdec_kernel: 2 parity blocks of kHdCtrl ints (hdec.cuh)
  uint32_t hcalls = 0;       // hdec_kernel calls on this workspace (parity)
  void* data = nullptr;
  size_t data_bytes = 0;
  cudaStream_t stream = nullptr;
  std::vector<void*> retired;  // outgrown data regions (freed by milo_stream_release)
};
std::mutex g_ws_mu;
long long* g_dbg = nullptr;  // milo_debug_timeline
int g_dbg_flags = 0;
std::map<std::pair<int, cudaStream_t>, DecodeWs> g_ws;
// One process-wide epoch counter (under g_ws_mu): a call's epoch is unique
// across every stream's workspace, so a word tagged by another stream's call
// can never pass for this call's.  0 (the control block's initial value) and
// 0xFFFFFFFF (the fill of fresh data regions) are never used; on wrap-around
// every workspace is re-initialised on its own stream before the epoch is reused.
uint32_t g_epoch = 0;

milo_status ws_init(DecodeWs& w, bool ctrl, bool data) {
  if (ctrl) CUDA_TRY(cudaMemsetAsync(w.ctrl, 0, kCtrlInts * 4, w.stream));
  if (ctrl && w.hctrl) {
    CUDA_TRY(cudaMemsetAsync(w.hctrl, 0, 2 * kHdCtrl * 4, w.stream));
    w.hcalls = 0;
  }
  if (data && w.data) CUDA_TRY(cudaMemsetAsync(w.data, 0xFF, w.data_bytes, w.stream));
  return MILO_OK;
}

milo_status next_epoch(int* epoch) {
  if (++g_epoch == 0xFFFFFFFFu) {
    for (auto& kv : g_ws) {
      int cur = 0;
      CUDA_TRY(cudaGetDevice(&cur));
      CUDA_TRY(cudaSetDevice(kv.first.first));
      const milo_status st = ws_init(kv.second, true, true);
      CUDA_TRY(cudaSetDevice(cur));
      if (st != MILO_OK) return st;
    }
    g_epoch = 1;
  }
  *epoch = (int)g_epoch;
  return MILO_OK;
}

// Returns the workspace of (device, stream) with >= data_bytes of data space and
// the epoch of this call.  Stream-ordered: fresh regions are filled with 0xFF
// (a tag no call carries) before the kernel that uses them; an outgrown region
// is retired, not freed, so a launch another host thread prepared with it
// cannot run after its release.
milo_status get_ws(cudaStream_t stream, size_t data_bytes, DecodeWs** out, int* epoch) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_ws_mu);
  DecodeWs& w = g_ws[{dev, stream}];
  w.stream = stream;
  if (!w.ctrl) {
    CUDA_TRY(cudaMalloc(&w.ctrl, kCtrlInts * 4));
    CUDA_TRY(cudaMemset(w.ctrl, 0, kCtrlInts * 4));
  }
  if (w.data_bytes < data_bytes) {
    if (w.data) w.retired.push_back(w.data);
    w.data = nullptr;
    w.data_bytes = 0;
    CUDA_TRY(cudaMallocAsync(&w.data, data_bytes, stream));
    w.data_bytes = data_bytes;
    const milo_status st = ws_init(w, false, true);
    if (st != MILO_OK) return st;
  }
  const milo_status st = next_epoch(epoch);
  if (st != MILO_OK) return st;
  *out = &w;
  return MILO_OK;
}

// Prefill workspace of (device, stream), grown on demand and reused (stream
// order makes reuse safe); kept apart from the decode workspace so no prefill
// bytes can alias the decode kernel's epoch-tagged words.  Outgrown regions are
// retired like the decode ones.
struct PfWs {
  void* mem = nullptr;
  size_t bytes = 0;
  std::vector<void*> retired;
};
std::map<std::pair<int, cudaStream_t>, PfWs> g_pf_ws;
milo_status get_pf_ws(cudaStream_t stream, size_t bytes, void** out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_ws_mu);
  auto& w = g_pf_ws[{dev, stream}];
  if (w.bytes < bytes) {
    const size_t cap = std::max(bytes, w.bytes + w.bytes / 4);
    if (w.mem) w.retired.push_back(w.mem);
    w.mem = nullptr;
    w.bytes = 0;
    CUDA_TRY(cudaMallocAsync(&w.mem, cap, stream));
    w.bytes = cap;
  }
  *out = w.mem;
  return MILO_OK;
}

// Frees every workspace this library keeps for (current device, stream): after
// the stream's pending work, the decode control block and data regions (also
// the retired ones) and the prefill region.
milo_status release_stream_ws(cudaStream_t stream) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_ws_mu);
  CUDA_TRY(cudaStreamSynchronize(stream));
  auto it = g_ws.find({dev, stream});
  if (it != g_ws.end()) {
    for (void* p : it->second.retired) CUDA_TRY(cudaFree(p));
    if (it->second.data) CUDA_TRY(cudaFree(it->second.data));
    if (it->second.ctrl) CUDA_TRY(cudaFree(it->second.ctrl));
    if (it->second.hctrl) CUDA_TRY(cudaFree(it->second.hctrl));
    g_ws.erase(it);
  }
  auto jt = g_pf_ws.find({dev, stream});
  if (jt != g_pf_ws.end()) {
    for (void* p : jt->second.retired) CUDA_TRY(cudaFree(p));
    if (jt->second.mem) CUDA_TRY(cudaFree(jt->second.mem));
    g_pf_ws.erase(jt);
  }
  return MILO_OK;
}

template <int NT, int NMAT1, bool MOE>
milo_status launch_decode(DecArgs a, const void* x, int32_t x_dtype, int64_t ldx, int nb_max,
                          int f_max, int r16_max, int64_t y_rows, cudaStream_t stream, int sms) {
  using CF = DecCfg<NT, NMAT1>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    CUDA_TRY(set_smem_min_carveout(decode_kernel<NT, NMAT1, MOE>, CF::kBytes));
    configured_dev = dev;
  }
  const int G = sms * CF::kCons;
  const int m_pad = CF::kMPad;
  Arena ar;
  const int64_t part_stride = CF::kPartMax;
  const size_t o_part = ar.take((size_t)2 * G * 2 * part_stride * 8);  // tagged (value, epoch) words
  const size_t o_t = ar.take((size_t)nb_max * 3 * m_pad * std::max(r16_max, 16) * 8);
  const size_t o_h = ar.take(MOE ? (size_t)nb_max * m_pad * f_max * 2 : 0);
  const size_t o_y = ar.take(MOE ? (size_t)y_rows * a.d * 4 : 0);
  // CTA-private binary16 copies of x (decode.cuh) when x is f32 (it is rounded
  // to binary16 on the way); binary16 x is read in place
  static const int xrep_env = [] {
    const char* e = getenv("MILO_XREP");
    return e ? atoi(e) : -1;
  }();
  const bool replicate = a.m <= 16 && (xrep_env >= 0 ? xrep_env == 1 : x_dtype == 0);
  const size_t o_x = ar.take(replicate ? (size_t)sms * a.m * a.d * 2
                                       : (x_dtype == 0 ? (size_t)a.m * a.d * 2 : 0));
  DecodeWs* w = nullptr;
  int epoch = 0;
  milo_status st = get_ws(stream, ar.size, &w, &epoch);
  if (st != MILO_OK) return st;
  uint8_t* base = static_cast<uint8_t*>(w->data);
  int32_t* c = w->ctrl;
  DecWs& W = a.ws;
  W.part = reinterpret_cast<uint64_t*>(base + o_part);
  W.t = reinterpret_cast<uint64_t*>(base + o_t);
  W.h = reinterpret_cast<__half*>(base + o_h);
  W.Y = reinterpret_cast<float*>(base + o_y);
  W.cnt1 = c;
  W.cnt2 = c + kCntCap;
  W.tcnt = W.cnt2 + kCntCap;
  W.bcnt = W.tcnt + kDecMaxBlocks * 3;
  W.ccnt = W.bcnt + kDecMaxBlocks;
  W.tflag = W.ccnt + kCCntCap;
  W.bflag = W.tflag + kDecMaxBlocks * 3;
  W.hflag = W.bflag + kDecMaxBlocks;
  if (MOE && (int64_t)nb_max * (f_max / 64) > kHflagCap) return fail(MILO_ERR_CONFIG, "decode: h flag capacity");
  {  // 32-bit stream-K range arithmetic: tiles of a phase x warps < 2^32 (decode.cuh rng_at)
    const int64_t kmax = std::max<int64_t>(a.d, f_max), nmax = std::max<int64_t>(a.d, f_max);
    const int64_t tiles_bound = (int64_t)nb_max * ((kmax / 32) * (nmax / 64) + (int64_t)(std::max(r16_max, 16) / 16) * 3 * (kmax / 32));
    if (tiles_bound * G >= (int64_t)1 << 32) return fail(MILO_ERR_CONFIG, "decode: too many tiles for one launch");
  }
  W.part_stride = part_stride;
  W.r16_max = std::max(r16_max, 16);
  W.f_max = f_max;
  a.epoch = epoch;
  a.gw = G;
  a.dbg = g_dbg;
  a.dbg_flags = g_dbg_flags;
  W.xrep = nullptr;
  a.x = x;
  a.x_dtype = x_dtype;
  a.ldx = ldx;
  if (replicate) {
    W.xrep = reinterpret_cast<__half*>(base + o_x);
  } else if (x_dtype == 0) {  // the kernel reads binary16 rows: round f32 rows once (gemm.cpp:144-146)
    __half* x16 = reinterpret_cast<__half*>(base + o_x);
    const int64_t n4 = (int64_t)a.m * (a.d / 4);
    const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)sms * 4);
    CUDA_TRY(launch(rows_to_half_kernel, dim3(std::max(grid, 1)), dim3(256), 0, stream, false,
                    static_cast<const float*>(x), (int64_t)a.m, (int64_t)a.d, ldx, x16));
    a.x = x16;
    a.x_dtype = 1;
    a.ldx = a.d;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(32 * CF::kWarps);
  cfg.dynamicSmemBytes = CF::kBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  ProfScope ps(kProfGemv1, stream);
  CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_kernel<NT, NMAT1, MOE>, a));
  return MILO_OK;
}

}  // namespace

extern "C" milo_status milo_stream_release(void* stream) {
  return release_stream_ws(static_cast<cudaStream_t>(stream));
}


// ---------------------------------------------------------------------------
// Prefill (tcgen05) path: activation images + pf_gemm_kernel.
// ---------------------------------------------------------------------------
namespace {

// token tile of the tcgen05 GEMM for a problem with `rows` tokens: 16 .. 128
int pf_ntok(int64_t rows) { return (int)std::min<int64_t>(kPfN, (rows + 15) / 16 * 16); }

int prefill_min_rows() {
  static const int v = [] {
    const char* e = getenv("MILO_PF_MIN");
    return e ? atoi(e) : 64;
  }();
  return v;
}

// Grouped activation images + LoRC t partials (pf_img_t_kernel), then the
// t hi / lo images (pf_t_images_kernel): one launch each per GEMM phase.
struct ImgTPlan {
  bool fuse_t = false;  // t partials in the image kernel (slower than pf_t_kernel for long k: off)
  std::vector<ImgJob> jobs;
  std::vector<TProb> tps;  // for pf_t_images_kernel (rows, rchunks, ks = k / 64, part, timg, ntok)
  int blocks = 0;
  void add(const void* x, int32_t x_dtype, int64_t ldx, const int32_t* row_ids, int64_t rows, int64_t k,
           int ntok, uint8_t* img, const milo_comp* const* comps, uint8_t* const* timg, float* const* part, int nc) {
    ImgJob J{};
    J.x = x;
    J.x_dtype = x_dtype;
    J.ldx = ldx;
    J.row_ids = row_ids;
    J.rows = (int32_t)rows;
    J.k = (int32_t)k;
    J.ntok = ntok;
    J.img = img;
    J.blk0 = blocks;
    for (int i = 0; i < nc; ++i) {
      const milo_comp* c = comps[i];
      if (!c || c->rank == 0 || !fuse_t) continue;
      ImgT& T = J.t[J.n_t++];
      T.ucodes = c->ucodes;
      T.uscales = c->uscales;
      T.ureal = c->ureal;
      T.rank = (int32_t)c->rank;
      T.gpr = c->gpr;
      T.rchunks = c->rch;
      T.part = part[i];
      TProb tp{};
      tp.rows = (int32_t)rows;
      tp.rchunks = c->rch;
      tp.ks = (int32_t)(k / kPfK);
      tp.part = part[i];
      tp.timg = timg[i];
      tp.ntok = ntok;
      tps.push_back(tp);
    }
    jobs.push_back(J);
    blocks += (int)(((rows + ntok - 1) / ntok) * (k / kPfK));
  }
  static size_t part_bytes(int64_t rows, int64_t k, const milo_comp* c, int sms) {
    if (!c || c->rank == 0) return 0;
    return (size_t)std::max<int64_t>(k / kPfK, t_splits(rows, k, c, sms)) * rows * c->rch * 64 * 4;
  }
  // k splits of pf_t_kernel: about kTCtasPerSm CTAs per SM over all `nprob` problems
  static int t_splits(int64_t rows, int64_t k, const milo_comp* c, int sms, int nprob = 1) {
    const int row_tiles = (int)((rows + kTRows - 1) / kTRows);
    return std::max(1, std::min<int>((int)(k / 256), (kTCtasPerSm * sms) / std::max(1, row_tiles * c->rch * nprob)));
  }
  // table: device memory for jobs + tps (>= table_bytes())
  size_t table_bytes() const { return ((jobs.size() * sizeof(ImgJob) + 255) & ~size_t(255)) + tps.size() * sizeof(TProb) + 256; }
  cudaError_t launch_all(uint8_t* table, cudaStream_t stream) const {
    if (jobs.empty()) return cudaSuccess;
    static thread_local int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
      cudaError_t e = cudaFuncSetAttribute(pf_img_t_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kImgTSmem);
      if (e != cudaSuccess) return e;
      configured_dev = dev;
    }
    const size_t jb = (jobs.size() * sizeof(ImgJob) + 255) & ~size_t(255);
    cudaError_t e = h2d_async(table, jobs.data(), jobs.size() * sizeof(ImgJob), stream);
    if (e != cudaSuccess) return e;
    if (!tps.empty()) {
      e = h2d_async(table + jb, tps.data(), tps.size() * sizeof(TProb), stream);
      if (e != cudaSuccess) return e;
    }
    e = fuse_t ? launch(pf_img_t_kernel<true>, dim3((unsigned)blocks), dim3(256), kImgTSmem, stream, false,
                        (const ImgJob*)table, (int)jobs.size(), (const int32_t*)nullptr)
               : launch(pf_img_t_kernel<false>, dim3((unsigned)blocks), dim3(256), 0, stream, false,
                        (const ImgJob*)table, (int)jobs.size(), (const int32_t*)nullptr);
    if (e != cudaSuccess || tps.empty()) return e;
    return launch(pf_t_images_kernel, dim3(256, (unsigned)tps.size()), dim3(256), 0, stream, false,
                  (const TProb*)(table + jb), (int)tps.size(), (const int32_t*)nullptr);
  }
};

// t = half(x) U for the prefill LoRC stages: pf_t_kernel (k split, fixed-order
// reduction) + pf_t_images_kernel; `table` holds the TProb array (device).
cudaError_t launch_t_batch(const std::vector<TProb>& v, int units, uint8_t* table, cudaStream_t stream) {
  if (v.empty()) return cudaSuccess;
  cudaError_t e = h2d_async(table, v.data(), v.size() * sizeof(TProb), stream);
  if (e != cudaSuccess) return e;
  bool coded = false, real = false;
  for (const TProb& t : v) (t.ucodes ? coded : real) = true;
  if (coded) e = launch(pf_t_kernel<0>, dim3(units), dim3(256), 0, stream, false, (const TProb*)table, (int)v.size(),
                        (const int32_t*)nullptr);
  if (e == cudaSuccess && real)
    e = launch(pf_t_kernel<1>, dim3(units), dim3(256), 0, stream, false, (const TProb*)table, (int)v.size(),
               (const int32_t*)nullptr);
  if (e != cudaSuccess) return e;
  return launch(pf_t_images_kernel, dim3(256, (unsigned)v.size()), dim3(256), 0, stream, false, (const TProb*)table,
                (int)v.size(), (const int32_t*)nullptr);
}
TProb make_tprob(const void* x, int32_t x_dtype, int64_t ldx, const int32_t* row_ids, int64_t rows, int64_t k,
                 int ntok, const milo_comp* c, uint8_t* timg, float* part, int sms, int unit0, int* units,
                 int nprob = 1) {
  TProb tp{};
  tp.x = x;
  tp.x_dtype = x_dtype;
  tp.ldx = ldx;
  tp.row_ids = row_ids;
  tp.rows = (int32_t)rows;
  tp.k = (int32_t)k;
  tp.rank = (int32_t)c->rank;
  tp.gpr = c->gpr;
  tp.rchunks = c->rch;
  tp.ks = ImgTPlan::t_splits(rows, k, c, sms, nprob);
  tp.ucodes = c->ucodes;
  tp.uscales = c->uscales;
  tp.ureal = c->ureal;
  tp.timg = timg;
  tp.part = part;
  tp.ntok = ntok;
  tp.unit0 = unit0;
  const int row_tiles = (int)((rows + kTRows - 1) / kTRows);
  *units = row_tiles * tp.rchunks * tp.ks;
  return tp;
}
cudaError_t launch_t(const void* x, int32_t x_dtype, int64_t ldx, const int32_t* row_ids, int64_t rows, int64_t k,
                     int ntok, const milo_comp* c, uint8_t* timg, float* part, uint8_t* table, int sms,
                     cudaStream_t stream) {
  int units = 0;
  std::vector<TProb> v{make_tprob(x, x_dtype, ldx, row_ids, rows, k, ntok, c, timg, part, sms, 0, &units)};
  return launch_t_batch(v, units, table, stream);
}

// NG = 2 n-tiles per item (activation images shared by two MMAs) when every
// problem's n is a multiple of 256 and the accumulators fit TMEM (one matrix).
template <int NMAT, int NG>
milo_status launch_prefill_ng(const PfProblem* host_probs, int n_probs, cudaStream_t stream, int sms,
                              uint8_t* scratch) {
  using CF = PfCfg<NMAT, NG>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    CUDA_TRY(set_smem(pf_gemm_kernel<NMAT, NG>, CF::kBytes));
    configured_dev = dev;
  }
  std::vector<int32_t> starts(n_probs + 1, 0);
  int ntok_max = 16;
  for (int i = 0; i < n_probs; ++i) {
    const PfProblem& P = host_probs[i];
    ntok_max = std::max(ntok_max, (int)P.ntok);
    starts[i + 1] = starts[i] + (P.n / (kPfM * NG)) * ((P.rows + P.ntok - 1) / P.ntok);
  }
  // problem table + starts travel in the scratch buffer (stream-ordered upload)
  const size_t pb = (size_t)n_probs * sizeof(PfProblem);
  CUDA_TRY(h2d_async(scratch, host_probs, pb, stream));
  CUDA_TRY(h2d_async(scratch + ((pb + 255) & ~size_t(255)), starts.data(), starts.size() * 4, stream));
  PfArgs a{};
  a.ntok_max = ntok_max;
  a.dbg = g_dbg;
  a.flags = g_dbg_flags;
  a.problems = reinterpret_cast<const PfProblem*>(scratch);
  a.item_start = reinterpret_cast<const int32_t*>(scratch + ((pb + 255) & ~size_t(255)));
  a.n_problems = n_probs;
  a.n_items = starts[n_probs];
  if (a.n_items == 0) return MILO_OK;
  static const int grid_cap = [] {  // experiments: MILO_PF_GRID caps the persistent grid
    const char* e = getenv("MILO_PF_GRID");
    return e ? atoi(e) : 0;
  }();
  const int grid = std::min(a.n_items, grid_cap > 0 ? std::min(grid_cap, sms) : sms);
  ProfScope ps(NMAT == 2 ? kProfGemv1 : kProfGemv2, stream);  // bench: w1|w3 (phase 1) / w2 or linear
  CUDA_TRY(launch(pf_gemm_kernel<NMAT, NG>, dim3(grid), dim3(PfRoles<NMAT, NG>::kThreads), CF::kBytes, stream, false, a));
  return MILO_OK;
}

int prefill_ng() {
  static const int v = [] {
    const char* e = getenv("MILO_PF_NG");
    return e ? atoi(e) : 2;
  }();
  return v;
}

template <int NMAT>
milo_status launch_prefill(const PfProblem* host_probs, int n_probs, cudaStream_t stream, int sms,
                           uint8_t* scratch) {
  // NG = 2 when it still fills the grid (it halves the item count)
  bool ng2 = NMAT == 1 && prefill_ng() == 2;
  int64_t items2 = 0;
  for (int i = 0; i < n_probs && ng2; ++i) {
    const PfProblem& P = host_probs[i];
    ng2 = P.n % (2 * kPfM) == 0;
    items2 += (P.n / (2 * kPfM)) * ((P.rows + P.ntok - 1) / P.ntok);
  }
  ng2 = ng2 && items2 >= sms;
  if (ng2) return launch_prefill_ng<1, 2>(host_probs, n_probs, stream, sms, scratch);
  return launch_prefill_ng<NMAT, 1>(host_probs, n_probs, stream, sms, scratch);
}

}  // namespace

// Debug hook (not in the public header): per-warp globaltimer stamps of the
// next decode launches, [grid warps][8] int64 on the device; NULL disables.
extern "C" void milo_debug_timeline(long long* dev_ptr) { g_dbg = dev_ptr; }
extern "C" void milo_debug_flags(int flags) { g_dbg_flags = flags; }

extern "C" milo_status milo_gemm_w3a16(const milo_weight* w, const milo_comp* comp,
                                       const milo_gemm_config* cfg, const void* A, int64_t m,
                                       int64_t a_cols, int32_t a_dtype, void* C, int32_t c_dtype,
                                       void* stream_) {
  if (!w || !cfg) return fail(MILO_ERR_ARGUMENT, "null argument");
  milo_status st = validate_gemm(w, comp, cfg, a_cols);
  if (st != MILO_OK) return st;
  if (m < 0) return fail(MILO_ERR_SHAPE, "negative row count");
  if (m == 0) return MILO_OK;
  if (!A || !C) return fail(MILO_ERR_ARGUMENT, "null A or C");
  if ((a_dtype != 0 && a_dtype != 1) || (c_dtype != 0 && c_dtype != 1))
    return fail(MILO_ERR_ARGUMENT, "unsupported dtype");
  DeviceProps props = device_props();
  if (!props.ok || props.major != 10) return fail(MILO_ERR_CUDA, "no sm_100 device");
  cudaStream_t stream = (cudaStream_t)stream_;

  const int nt = m <= 8 ? 1 : 2;
  const int m_pad = 8 * nt;
  const int64_t k = (int64_t)w->rows, n = (int64_t)w->cols;
  const bool pf_comp_ok = !(comp && comp->rank > 0) || comp->vimg != nullptr;
  // (the prefill kernel's producers move 128 k per ring slot)
  if (!legacy_path() && m >= prefill_min_rows() && n % kPfM == 0 && k % (2 * kPfK) == 0 && pf_comp_ok) {
    // tcgen05 path: activation images (binary16, SW128) then the grouped GEMM
    const int ntok = pf_ntok(m);
    const int64_t tiles = (m + ntok - 1) / ntok, ks = k / kPfK;
    void* mem = nullptr;
    const size_t img_b = (size_t)tiles * ks * ntok * 128;
    const bool lorc = comp && comp->rank > 0;
    const size_t t_img_b = lorc ? (size_t)tiles * comp->rch * 2 * ntok * 128 : 0;
    const size_t t_part_b = ImgTPlan::part_bytes(m, k, lorc ? comp : nullptr, props.sms);
    CUDA_TRY(cudaMallocAsync(&mem, img_b + t_img_b + t_part_b + 16384, stream));
    uint8_t* img = static_cast<uint8_t*>(mem);
    uint8_t* timg = img + img_b;
    float* tpart = reinterpret_cast<float*>(img + img_b + t_img_b);
    uint8_t* tabs = img + img_b + t_img_b + t_part_b;  // [GEMM problems | image plan @8K | t table @12K]
    PfProblem P{};
    P.w[0] = w->tiles;
    P.act = img;
    P.k = (int32_t)k;
    P.n = (int32_t)n;
    P.rows = (int32_t)m;
    P.ntok = ntok;
    P.mode = w->mode;
    P.kind = 0;
    P.out_dtype = c_dtype;
    P.ldo = n;
    P.out = C;
    if (lorc) {
      P.vimg[0] = comp->vimg;
      P.timg[0] = timg;
      P.rchunks[0] = comp->rch;
    }
    // two passes like moe_prefill: the tables go up before the first kernel
    auto sequence = [&]() -> milo_status {
      ImgTPlan plan;
      const milo_comp* cs[1] = {comp};
      plan.add(A, a_dtype, a_cols, nullptr, m, k, ntok, img, cs, &timg, &tpart, 1);
      cudaError_t e = plan.launch_all(tabs + 8192, stream);
      if (e == cudaSuccess && lorc)
        e = launch_t(A, a_dtype, a_cols, nullptr, m, k, ntok, comp, timg, tpart, tabs + 12288, props.sms, stream);
      if (e != cudaSuccess) return fail(MILO_ERR_CUDA, "launch failed: %s", cudaGetErrorString(e));
      return launch_prefill<1>(&P, 1, stream, props.sms, tabs);
    };
    {
      struct PassReset {
        ~PassReset() {
          g_dry = false;
          g_pin.mode = 0;
          g_pin.rec.clear();
          g_pin.lo = g_pin.hi = nullptr;
        }
      } pass_reset;
      pin_begin();
      g_pin.lo = tabs;
      g_pin.hi = tabs + 16384;
      g_pin.mode = 1;
      g_dry = true;
      st = sequence();
      g_dry = false;
      g_pin.mode = 0;
      if (st == MILO_OK) {
        cudaError_t e = pin_flush(stream);
        if (e != cudaSuccess) st = fail(MILO_ERR_CUDA, "upload failed: %s", cudaGetErrorString(e));
      }
      if (st == MILO_OK) {
        g_pin.mode = 2;
        st = sequence();
      }
    }
    pin_end(stream);
    cudaFreeAsync(mem, stream);
    return st;
  }
  if (!legacy_path()) {
    DecArgs a{};
    a.moe = 0;
    a.lin.m[0] = make_decmat(w, comp);
    a.d = (int32_t)k;
    a.out_dtype = c_dtype;
    a.ldo = n;
    const int r16 = a.lin.m[0].r16;
    const int64_t per_block_slabs = n / 64 + r16 / 16;
    const int64_t max_blocks =
        std::max<int64_t>(1, std::min<int64_t>(DecCfg<1, 1>::kMaxBlocks, kCntCap / per_block_slabs));
    const size_t xs = a_dtype == 0 ? 4 : 2, cs = c_dtype == 0 ? 4 : 2;
    for (int64_t done = 0; done < m;) {
      const int64_t mm = std::min<int64_t>(m - done, max_blocks * m_pad);
      a.m = (int32_t)mm;
      const void* xa = static_cast<const uint8_t*>(A) + done * a_cols * xs;
      a.out = static_cast<uint8_t*>(C) + done * n * cs;
      const int nb = (int)((mm + m_pad - 1) / m_pad);
      st = nt == 1 ? launch_decode<1, 1, false>(a, xa, a_dtype, a_cols, nb, 0, r16, 0, stream, props.sms)
                   : launch_decode<2, 1, false>(a, xa, a_dtype, a_cols, nb, 0, r16, 0, stream, props.sms);
      if (st != MILO_OK) return st;
      done += mm;
    }
    return MILO_OK;
  }
  const int rank = (comp && comp->rank > 0) ? (int)comp->rank : 0;
  int64_t done = 0;
  while (done < m) {
    const int64_t mm = std::min<int64_t>(m - done, (int64_t)(kMaxProblems - 1) * m_pad);
    const int blocks = (int)((mm + m_pad - 1) / m_pad);
    const int64_t slabs = (int64_t)blocks * (n / 64);
    Arena ar;
    const int64_t act_block_words = (k / 32) * m_pad * 16;
    const size_t o_act = ar.take((size_t)blocks * act_block_words * 4);
    const size_t o_prob = ar.take((size_t)blocks * sizeof(GemvProblem));
    const size_t o_np = ar.take(4);
    const size_t o_t = ar.take((size_t)blocks * m_pad * std::max(rank, 1) * 4);
    const size_t ws_b = nt == 1 ? GroupedWs<1, 1>::ws_bytes(props.sms) : GroupedWs<2, 1>::ws_bytes(props.sms);
    const size_t full_b = nt == 1 ? GroupedWs<1, 1>::full_bytes(slabs) : GroupedWs<2, 1>::full_bytes(slabs);
    const size_t part_b = nt == 1 ? GroupedWs<1, 1>::lorc_bytes(blocks, k, rank)
                                  : GroupedWs<2, 1>::lorc_bytes(blocks, k, rank);
    const size_t o_ws = ar.take(ws_b);
    const size_t o_full = ar.take(full_b);
    const size_t o_part = ar.take(part_b);
    const size_t o_tc = ar.take((size_t)blocks * 2 * 4);
    const size_t o_sc = ar.take((size_t)slabs * 4);
    void* mem = nullptr;
    CUDA_TRY(cudaMallocAsync(&mem, ar.size, stream));
    uint8_t* base = static_cast<uint8_t*>(mem);

    GemvProblem tmpl{};
    tmpl.w[0] = w->tiles;
    tmpl.k = (int32_t)k;
    tmpl.n = (int32_t)n;
    tmpl.mode = w->mode;
    tmpl.kind = kStoreRows;
    tmpl.out_dtype = c_dtype;
    tmpl.ldo = n;
    tmpl.out = c_dtype == 0 ? (void*)(static_cast<float*>(C) + done * n)
                            : (void*)(static_cast<__half*>(C) + done * n);
    if (rank > 0) {
      fill_comp(tmpl, 0, comp);
      tmpl.t[0] = reinterpret_cast<float*>(base + o_t);
    }
    LinearPrep lp{};
    lp.A = a_dtype == 0 ? (const void*)(static_cast<const float*>(A) + done * a_cols)
                        : (const void*)(static_cast<const __half*>(A) + done * a_cols);
    lp.m = mm;
    lp.k = k;
    lp.lda = a_cols;
    lp.a_dtype = a_dtype;
    lp.m_pad = m_pad;
    lp.n_blocks = blocks;
    lp.act = reinterpret_cast<uint32_t*>(base + o_act);
    lp.tmpl = tmpl;
    lp.act_block_words = act_block_words;
    lp.t_block_floats = (int64_t)m_pad * rank;
    lp.out_block_elems = (int64_t)m_pad * n;
    lp.problems = reinterpret_cast<GemvProblem*>(base + o_prob);
    lp.n_problems = reinterpret_cast<int32_t*>(base + o_np);
    lp.counters = reinterpret_cast<int32_t*>(base + o_sc);
    lp.n_counters = (int32_t)slabs;
    lp.t_counters = reinterpret_cast<int32_t*>(base + o_tc);
    lp.n_t_counters = blocks * 2;
    const int64_t prep_threads = (int64_t)blocks * m_pad * (k / 2);
    const int prep_grid = (int)std::min<int64_t>((prep_threads + 255) / 256, props.sms * 8);
    cudaError_t e = launch(prep_linear_kernel, dim3(prep_grid), dim3(256), 0, stream, false, lp);
    if (e != cudaSuccess) {
      cudaFreeAsync(mem, stream);
      return fail(MILO_ERR_CUDA, "launch failed: %s", cudaGetErrorString(e));
    }
    float* ws = reinterpret_cast<float*>(base + o_ws);
    float* full = reinterpret_cast<float*>(base + o_full);
    float* part = reinterpret_cast<float*>(base + o_part);
    int32_t* tc = lp.t_counters;
    st = nt == 1 ? run_grouped<1, 1>(lp.problems, lp.n_problems, blocks, slabs, k, rank, ws, full,
                                     lp.counters, part, tc, stream, props.sms, kProfGemv1)
                 : run_grouped<2, 1>(lp.problems, lp.n_problems, blocks, slabs, k, rank, ws, full,
                                     lp.counters, part, tc, stream, props.sms, kProfGemv1);
    cudaFreeAsync(mem, stream);
    if (st != MILO_OK) return st;
    done += mm;
  }
  return MILO_OK;
}

extern "C" milo_status milo_gemm_w3a16_host(const milo_weight* w, const milo_comp* comp,
                                            const milo_gemm_config* cfg, const float* A,
                                            int64_t m, int64_t a_cols, float* C) {
  if (!w || !cfg) return fail(MILO_ERR_ARGUMENT, "null argument");
  milo_status st = validate_gemm(w, comp, cfg, a_cols);
  if (st != MILO_OK) return st;
  if (m <= 0) return m == 0 ? MILO_OK : fail(MILO_ERR_SHAPE, "negative row count");
  cudaStream_t stream = nullptr;
  void *dA = nullptr, *dC = nullptr;
  const size_t abytes = (size_t)m * a_cols * 4, cbytes = (size_t)m * w->cols * 4;
  CUDA_TRY(cudaMallocAsync(&dA, abytes, stream));
  CUDA_TRY(cudaMallocAsync(&dC, cbytes, stream));
  CUDA_TRY(cudaMemcpyAsync(dA, A, abytes, cudaMemcpyHostToDevice, stream));
  st = milo_gemm_w3a16(w, comp, cfg, dA, m, a_cols, MILO_F32, dC, MILO_F32, stream);
  if (st == MILO_OK) {
    cudaError_t e = cudaMemcpyAsync(C, dC, cbytes, cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) st = fail(MILO_ERR_CUDA, "copy back failed: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(dA, stream);
  cudaFreeAsync(dC, stream);
  cudaError_t e = cudaStreamSynchronize(stream);
  if (st == MILO_OK && e != cudaSuccess) st = fail(MILO_ERR_CUDA, "%s", cudaGetErrorString(e));
  return st;
}

// ---------------------------------------------------------------------------
// MoE layer
// ---------------------------------------------------------------------------
struct milo_moe {
  int32_t E = 0, n_shared = 0, K = 0, score_mode = 0;
  int32_t d = 0, f_max = 0, rank1_max = 0, rank2_max = 0;
  ExpertDev* dev_experts = nullptr;  // E + n_shared entries
  DecExpert* dec_experts = nullptr;  // decode-kernel view of the same experts
  int32_t r16_max = 0;
  // prefill view: per expert, per matrix (w1, w3, w2) weight tiles + compensator
  std::vector<std::array<const milo_weight*, 3>> hw;
  std::vector<std::array<const milo_comp*, 3>> hc;
  bool prefill_ok = true;
  // host-buffer entry point: pinned staging (x | logits, then out) and device buffer, grown on demand
  void* host_stage = nullptr;
  void* dev_stage = nullptr;
  size_t stage_bytes = 0;
  std::mutex stage_mu;  // the staging is per handle; handles may be shared across threads
  __half* gate = nullptr;  // optional router gate, E x d binary16 (milo_moe_set_gate)
  PfExpertStatic* pf_static = nullptr;  // device: per expert, what moe_plan_kernel needs
  int t_kinds[2] = {0, 0};               // per phase: bit 0 symm-INT3 factors, bit 1 real factors
  int32_t rch_max[3] = {0, 0, 0};       // largest 64-rank chunk count per matrix
  bool hd_ok = true;                    // hdec_kernel eligible (int3 / no compensators, 64-multiple shapes)
  HdExp* hd_exp = nullptr;              // device: hdec_kernel's per-expert static view
  uint8_t* hd_w2maps = nullptr;         // device: per expert, a 128-byte TMA map of W2's tiles
};

extern "C" milo_status milo_moe_create(const milo_expert_desc* experts, int32_t n_experts,
                                       const milo_expert_desc* shared, int32_t n_shared,
                                       int32_t top_k, int32_t score_mode, milo_moe** out) {
  if (!out) return fail(MILO_ERR_ARGUMENT, "null out");
  *out = nullptr;
  if (n_experts < 0 || n_shared < 0 || n_experts + n_shared <= 0 ||
      n_experts + n_shared > kRouteMaxE)
    return fail(MILO_ERR_CONFIG, "need 1..%d experts", kRouteMaxE);
  if (n_experts > 0 && (top_k < 1 || top_k > 16 || top_k > n_experts))
    return fail(MILO_ERR_CONFIG, "top_k must be in [1, min(16, n_experts)]");
  if (score_mode != 0 && score_mode != 1) return fail(MILO_ERR_CONFIG, "unknown score mode");
  std::vector<ExpertDev> host(n_experts + n_shared);
  std::vector<DecExpert> dhost(n_experts + n_shared);
  auto* moe = new milo_moe();
  moe->E = n_experts;
  moe->n_shared = n_shared;
  moe->K = n_experts > 0 ? top_k : 0;
  moe->score_mode = score_mode;
  for (int i = 0; i < n_experts + n_shared; ++i) {
    const milo_expert_desc& ex = i < n_experts ? experts[i] : shared[i - n_experts];
    const milo_weight* w[3] = {ex.w1, ex.w3, ex.w2};
    const milo_comp* c[3] = {ex.c1, ex.c3, ex.c2};
    for (int j = 0; j < 3; ++j)
      if (!w[j] || !w[j]->tiles) {
        delete moe;
        return fail(MILO_ERR_CONFIG, "expert %d matrix %d has no device layout", i, j);
      }
    const uint64_t d = w[0]->rows, f = w[0]->cols;
    if (w[1]->rows != d || w[1]->cols != f || w[2]->rows != f || w[2]->cols != d) {
      delete moe;
      return fail(MILO_ERR_SHAPE, "expert %d: need w1,w3 d x f and w2 f x d", i);
    }
    if (moe->d == 0) moe->d = (int32_t)d;
    if ((int32_t)d != moe->d) {
      delete moe;
      return fail(MILO_ERR_SHAPE, "expert %d: hidden size differs", i);
    }
    if (w[0]->mode != w[1]->mode) {
      delete moe;
      return fail(MILO_ERR_CONFIG, "expert %d: w1 and w3 modes differ", i);
    }
    ExpertDev& e = host[i];
    moe->hw.push_back({w[0], w[1], w[2]});
    moe->hc.push_back({c[0], c[1], c[2]});
    for (int j = 0; j < 3; ++j) {
      const bool comp_ok = !(c[j] && c[j]->rank > 0) || c[j]->vimg != nullptr;
      if (w[j]->cols % kPfM != 0 || w[j]->rows % (2 * kPfK) != 0 || !comp_ok) moe->prefill_ok = false;
    }
    for (int j = 0; j < 3; ++j) {
      const bool has_c = c[j] && c[j]->rank > 0;
      if ((has_c && (c[j]->storage != 1 || !c[j]->upt)) || w[j]->rows % 64 != 0 || w[j]->cols % 64 != 0)
        moe->hd_ok = false;
    }
    for (int j = 0; j < 3; ++j) {
      dhost[i].m[j] = make_decmat(w[j], c[j]);
      moe->r16_max = std::max(moe->r16_max, dhost[i].m[j].r16);
    }
    e.f = (int32_t)f;
    e.mode = w[0]->mode;
    moe->f_max = std::max(moe->f_max, (int32_t)f);
    for (int j = 0; j < 3; ++j) {
      e.w[j] = w[j]->tiles;
      if (j == 2 && w[2]->mode != w[0]->mode) {
        delete moe;
        return fail(MILO_ERR_CONFIG, "expert %d: w2 mode differs", i);
      }
      if (c[j] && c[j]->rank > 0) {
        if (c[j]->rows != w[j]->rows || c[j]->cols != w[j]->cols) {
          delete moe;
          return fail(MILO_ERR_SHAPE, "expert %d: compensator %d shape mismatch", i, j);
        }
        e.rank[j] = (int32_t)c[j]->rank;
        e.gpr[j] = c[j]->gpr;
        e.ucodes[j] = c[j]->ucodes;
        e.uscales[j] = c[j]->uscales;
        e.ureal[j] = c[j]->ureal;
        e.vcodes[j] = c[j]->vcodes;
        e.vscales[j] = c[j]->vscales;
        e.vreal[j] = c[j]->vreal;
        if (j < 2) moe->rank1_max = std::max(moe->rank1_max, e.rank[j]);
        else moe->rank2_max = std::max(moe->rank2_max, e.rank[j]);
      }
    }
  }
  cudaError_t err = cudaMalloc(&moe->dev_experts, host.size() * sizeof(ExpertDev));
  if (err == cudaSuccess)
    err = cudaMemcpy(moe->dev_experts, host.data(), host.size() * sizeof(ExpertDev),
                     cudaMemcpyHostToDevice);
  if (err == cudaSuccess) err = cudaMalloc(&moe->dec_experts, dhost.size() * sizeof(DecExpert));
  if (err == cudaSuccess)
    err = cudaMemcpy(moe->dec_experts, dhost.data(), dhost.size() * sizeof(DecExpert),
                     cudaMemcpyHostToDevice);
  {  // hdec_kernel's per-expert static view
    std::vector<HdExp> hx(dhost.size());
    for (size_t i = 0; i < dhost.size(); ++i) {
      const DecExpert& X = dhost[i];
      hx[i].nu = X.m[0].n / 64;
      hx[i].kt2 = X.m[0].n / 32;
      hx[i].mode = (int8_t)X.m[0].mode;
      for (int j = 0; j < 3; ++j) {
        const int nks = X.m[j].rank > 0 ? X.m[j].r16 / 16 : 0;
        if (nks > 127) moe->hd_ok = false;
        hx[i].nks[j] = (int8_t)std::min(nks, 127);
        hx[i].gpr[j] = (int8_t)X.m[j].gpr;
      }
    }
    if (err == cudaSuccess) err = cudaMalloc(&moe->hd_exp, hx.size() * sizeof(HdExp));
    if (err == cudaSuccess) err = cudaMemcpy(moe->hd_exp, hx.data(), hx.size() * sizeof(HdExp), cudaMemcpyHostToDevice);
    // W2 of every expert as a 2D tensor of u64: rows = 64-column slabs, columns = the
    // slab's k-run (f / 32 tiles x 112 u64); boxes of 8 slabs x 2 k-tiles feed a P2 stage
    std::vector<CUtensorMap> maps(dhost.size());
    for (size_t i = 0; i < dhost.size() && moe->hd_ok; ++i) {
      const DecMat& M = dhost[i].m[2];
      const cuuint64_t kt2 = (cuuint64_t)M.k / 32, nslabs = (cuuint64_t)M.n / 64;
      const cuuint64_t dims[2] = {kt2 * 112, nslabs};
      const cuuint64_t strides[1] = {kt2 * 896};
      const cuuint32_t box[2] = {224, (cuuint32_t)kW2Box};
      const cuuint32_t estr[2] = {1, 1};
      // the driver entry point is resolved at run time: no link-time libcuda dependency
      using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
      static EncodeFn encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
          fn = nullptr;
        return reinterpret_cast<EncodeFn>(fn);
      }();
      const CUresult r = encode ? encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, (void*)M.w, dims, strides, box,
                                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                                : CUDA_ERROR_NOT_SUPPORTED;
      if (r != CUDA_SUCCESS) moe->hd_ok = false;  // the h-local kernel needs the map
    }
    static_assert(sizeof(CUtensorMap) == 128, "tensor map size");
    if (err == cudaSuccess) err = cudaMalloc(&moe->hd_w2maps, maps.size() * 128);
    if (err == cudaSuccess) err = cudaMemcpy(moe->hd_w2maps, maps.data(), maps.size() * 128, cudaMemcpyHostToDevice);
  }
  {  // the prefill planner's static view (moe_plan_kernel)
    std::vector<PfExpertStatic> ps(host.size());
    for (size_t i = 0; i < host.size(); ++i)
      for (int j = 0; j < 3; ++j) {
        const milo_weight* w = moe->hw[i][j];
        const milo_comp* c = moe->hc[i][j];
        PfMatStatic& M = ps[i].m[j];
        M.w = w->tiles;
        M.k = (int32_t)w->rows;
        M.n = (int32_t)w->cols;
        M.mode = w->mode;
        if (c && c->rank > 0) {
          M.vimg = c->vimg;
          M.ucodes = c->ucodes;
          M.uscales = c->uscales;
          M.ureal = c->ureal;
          M.rank = (int32_t)c->rank;
          M.gpr = c->gpr;
          M.rch = c->rch;
          moe->rch_max[j] = std::max(moe->rch_max[j], c->rch);
          moe->t_kinds[j == 2 ? 1 : 0] |= c->ucodes ? 1 : 2;
        }
      }
    if (err == cudaSuccess) err = cudaMalloc(&moe->pf_static, ps.size() * sizeof(PfExpertStatic));
    if (err == cudaSuccess)
      err = cudaMemcpy(moe->pf_static, ps.data(), ps.size() * sizeof(PfExpertStatic), cudaMemcpyHostToDevice);
  }
  if (err != cudaSuccess) {
    cudaFree(moe->dev_experts);
    cudaFree(moe->dec_experts);
    cudaFree(moe->pf_static);
    cudaFree(moe->hd_exp);
    cudaFree(moe->hd_w2maps);
    delete moe;
    return fail(MILO_ERR_CUDA, "expert table upload failed: %s", cudaGetErrorString(err));
  }
  *out = moe;
  return MILO_OK;
}

extern "C" milo_status milo_moe_destroy(milo_moe* moe) {
  if (!moe) return MILO_OK;
  cudaFree(moe->dev_experts);
  cudaFree(moe->dec_experts);
  cudaFree(moe->pf_static);
  cudaFree(moe->hd_exp);
  cudaFree(moe->hd_w2maps);
  if (moe->host_stage) cudaFreeHost(moe->host_stage);
  if (moe->dev_stage) cudaFree(moe->dev_stage);
  if (moe->gate) cudaFree(moe->gate);
  delete moe;
  return MILO_OK;
}

extern "C" milo_status milo_router_topk(const float* logits, int64_t m, int32_t E, int32_t K,
                                        int32_t score_mode, int32_t* ids, float* w,
                                        void* stream) {
  if (m < 0 || E < 1 || K < 1 || K > 16 || K > E) return fail(MILO_ERR_CONFIG, "bad router shape");
  if (m == 0) return MILO_OK;
  if (!logits || !ids || !w) return fail(MILO_ERR_ARGUMENT, "null argument");
  const int warps = 8;
  CUDA_TRY(launch(router_topk_kernel, dim3((unsigned)((m + warps - 1) / warps)), dim3(32 * warps),
                  0, (cudaStream_t)stream, true, logits, m, E, K, score_mode, ids, w));
  return MILO_OK;
}

namespace {

template <int NT>
milo_status moe_run(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype,
                    const float* logits, int32_t* ids, float* wts, void* out, int32_t out_dtype,
                    cudaStream_t stream, int sms) {
  constexpr int m_pad = 8 * NT;
  const int K = moe->K, E = moe->E, S = moe->n_shared;
  const int64_t d = moe->d, f_max = moe->f_max;
  const int64_t blocks_max = std::min<int64_t>(
      kMaxProblems - 1, (m * K + m_pad - 1) / m_pad + std::min<int64_t>(E, m * K) +
                            (int64_t)S * ((m + m_pad - 1) / m_pad));
  const int r1 = moe->rank1_max, r2 = moe->rank2_max;
  const int64_t slabs1 = blocks_max * (f_max / 64), slabs2 = blocks_max * (d / 64);
  Arena ar;
  const size_t o_elist = ar.take((size_t)(m * K + S * m + 1) * 4);
  const size_t o_bexp = ar.take((size_t)blocks_max * 4);
  const size_t o_bst = ar.take((size_t)blocks_max * 4);
  const size_t o_p1 = ar.take((size_t)blocks_max * sizeof(GemvProblem));
  const size_t o_p2 = ar.take((size_t)blocks_max * sizeof(GemvProblem));
  const size_t o_np = ar.take(16);
  const int64_t act_block = (d / 32) * m_pad * 64;
  const int64_t h_block = (f_max / 32) * m_pad * 64;
  const size_t o_act = ar.take((size_t)blocks_max * act_block);
  const size_t o_h = ar.take((size_t)blocks_max * h_block);
  const size_t o_t1 = ar.take((size_t)blocks_max * 2 * m_pad * std::max(r1, 1) * 4);
  const size_t o_t2 = ar.take((size_t)blocks_max * m_pad * std::max(r2, 1) * 4);
  const size_t o_pa1 = ar.take(GroupedWs<NT, 2>::lorc_bytes(blocks_max, d, r1));
  const size_t o_pa2 = ar.take(GroupedWs<NT, 1>::lorc_bytes(blocks_max, f_max, r2));
  const size_t o_ws = ar.take(std::max(GroupedWs<NT, 2>::ws_bytes(sms), GroupedWs<NT, 1>::ws_bytes(sms)));
  const size_t o_full1 = ar.take(GroupedWs<NT, 2>::full_bytes(slabs1));
  const size_t o_full2 = ar.take(GroupedWs<NT, 1>::full_bytes(slabs2));
  const int64_t n_zero = 4 * blocks_max + slabs1 + slabs2;  // lorc + slab fix-up counters
  const size_t o_zero = ar.take((size_t)n_zero * 4);
  const size_t o_Y = ar.take((size_t)(m * K + S * m) * d * 4);
  void* mem = nullptr;
  CUDA_TRY(cudaMallocAsync(&mem, ar.size, stream));
  uint8_t* base = static_cast<uint8_t*>(mem);
  int32_t* np = reinterpret_cast<int32_t*>(base + o_np);
  int32_t* zero = reinterpret_cast<int32_t*>(base + o_zero);
  int32_t* tc1 = zero;
  int32_t* tc2 = tc1 + 2 * blocks_max;
  int32_t* sc1 = tc2 + 2 * blocks_max;
  int32_t* sc2 = sc1 + slabs1;

  MoeRouteArgs ra{};
  ra.ids = ids;
  ra.m = m;
  ra.K = K;
  ra.E = E;
  ra.n_shared = S;
  ra.d = (int32_t)d;
  ra.m_pad = m_pad;
  ra.experts = moe->dev_experts;
  ra.max_blocks = (int32_t)blocks_max;
  ra.elist = reinterpret_cast<int32_t*>(base + o_elist);
  ra.block_expert = reinterpret_cast<int32_t*>(base + o_bexp);
  ra.block_start = reinterpret_cast<int32_t*>(base + o_bst);
  ra.p1 = reinterpret_cast<GemvProblem*>(base + o_p1);
  ra.p2 = reinterpret_cast<GemvProblem*>(base + o_p2);
  ra.n_p1 = np;
  ra.n_p2 = np + 1;
  ra.n_blocks_out = np + 2;
  ra.act_pool = base + o_act;
  ra.h_pool = base + o_h;
  ra.h_block_bytes = h_block;
  ra.t1_pool = reinterpret_cast<float*>(base + o_t1);
  ra.t2_pool = reinterpret_cast<float*>(base + o_t2);
  ra.rank1_max = std::max(r1, 1);
  ra.rank2_max = std::max(r2, 1);
  ra.Y = reinterpret_cast<float*>(base + o_Y);
  ra.zero_ptr = zero;
  ra.zero_count = n_zero;
  ra.logits = logits;
  ra.ids_out = ids;
  ra.wts_out = wts;
  ra.score_mode = moe->score_mode;
  milo_status st = MILO_OK;
  const int route_threads = (int)std::min<int64_t>(kRouteThreads, std::max<int64_t>(128, (m + 31) / 32 * 32));
  cudaError_t e = launch(moe_route_kernel, dim3(1), dim3(route_threads), 0, stream, true, ra);
  if (e == cudaSuccess)
    e = launch(moe_gather_kernel, dim3((unsigned)blocks_max, m_pad), dim3(128), 0, stream, true, x,
               x_dtype, d, K, m, (const int32_t*)ra.elist, (const int32_t*)ra.block_start,
               (const int32_t*)ra.block_expert, (const int32_t*)ra.n_p1, E, m_pad, ra.act_pool,
               (const GemvProblem*)ra.p1);
  if (e != cudaSuccess) st = fail(MILO_ERR_CUDA, "launch failed: %s", cudaGetErrorString(e));
  float* ws = reinterpret_cast<float*>(base + o_ws);
  if (st == MILO_OK)
    st = run_grouped<NT, 2>(ra.p1, ra.n_p1, blocks_max, slabs1, d, r1, ws,
                            reinterpret_cast<float*>(base + o_full1), sc1,
                            reinterpret_cast<float*>(base + o_pa1), tc1, stream, sms, kProfGemv1);
  if (st == MILO_OK)
    st = run_grouped<NT, 1>(ra.p2, ra.n_p2, blocks_max, slabs2, f_max, r2, ws,
                            reinterpret_cast<float*>(base + o_full2), sc2,
                            reinterpret_cast<float*>(base + o_pa2), tc2, stream, sms, kProfGemv2);
  if (st == MILO_OK) {
    const int64_t total = m * (d / 4);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
    e = launch(moe_combine_kernel, dim3(grid), dim3(256), 0, stream, true,
               (const float*)ra.Y, ids, wts, m, K, S, d, out, out_dtype);
    if (e != cudaSuccess) st = fail(MILO_ERR_CUDA, "launch failed: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(mem, stream);
  return st;
}

}  // namespace

namespace {

// Prefill MoE layer on the tcgen05 GEMM (m > 16 tokens): routing on the device,
// one host synchronization to plan the grouped GEMMs (per-expert token lists in
// ascending token order), then per phase: activation images, t = x U, the
// grouped W3A16 + LoRC GEMM (phase 1 with SwiGLU), and the weighted combine.
milo_status moe_prefill(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype, const float* logits,
                        int32_t* ids, float* wts, void* out, int32_t out_dtype, cudaStream_t stream, int sms) {
  const int E = moe->E, K = moe->K, S = moe->n_shared;
  const int64_t d = moe->d;
  static const bool host_prof = getenv("MILO_HOST_PROF") != nullptr;  // experiments: host phase times
  auto hnow = [] { return std::chrono::steady_clock::now(); };
  const auto h0 = hnow();
  auto hmark = [&](const char* what) {
    if (host_prof)
      std::fprintf(stderr, "moe_prefill host %-12s %8.1f us\n", what,
                   std::chrono::duration<double, std::micro>(hnow() - h0).count());
  };
  if (K > 0 && logits) {
    CUDA_TRY(launch(router_topk_kernel, dim3((unsigned)((m + 7) / 8)), dim3(256), 0, stream, false, logits, m, E,
                    K, moe->score_mode, ids, wts));
  }
  // ---- plan on the host (the reference composition order)
  std::vector<int32_t> hids((size_t)m * std::max(K, 1));
  if (K > 0) {
    // routing ids to the host: a one-CTA kernel writes them into mapped pinned
    // memory followed by this call's epoch in a flag word, and the host spins on
    // the flag (no D2H copy launch, no synchronise wake-up on the critical path)
    static thread_local int32_t* pin_ids = nullptr;  // [cap ids | flag]
    static thread_local size_t pin_ids_n = 0;
    static thread_local int32_t pub_epoch = 0;
    if (pin_ids_n < hids.size()) {
      if (pin_ids) cudaFreeHost(pin_ids);
      pin_ids = nullptr;
      pin_ids_n = 0;
      const size_t cap = std::max<size_t>(hids.size(), 4096);
      CUDA_TRY(cudaMallocHost(&pin_ids, (cap + 32) * 4));
      pin_ids_n = cap;
      pin_ids[cap] = 0;
    }
    volatile int32_t* flag = pin_ids + pin_ids_n;
    pub_epoch = pub_epoch == INT32_MAX ? 1 : pub_epoch + 1;
    const int32_t ep = pub_epoch;
    int32_t* d_pin = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_pin), pin_ids, 0));
    CUDA_TRY(launch(publish_ids_kernel, dim3(1), dim3(256), 0, stream, false, (const int32_t*)ids,
                    (int64_t)hids.size(), d_pin, (volatile int32_t*)(d_pin + pin_ids_n), ep));
    for (uint32_t it = 1; *flag != ep; ++it) {
      if ((it & 4095) == 0) {  // a failed stream never publishes: check it now and then
        const cudaError_t q = cudaStreamQuery(stream);
        if (q != cudaErrorNotReady && q != cudaSuccess) return fail(MILO_ERR_CUDA, "%s", cudaGetErrorString(q));
        if (q == cudaSuccess && *flag != ep) return fail(MILO_ERR_CUDA, "prefill: routing ids not published");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    std::memcpy(hids.data(), pin_ids, hids.size() * 4);
  }
  hmark("ids synced");
  struct Grp { int e; int64_t off, rows; };
  std::vector<Grp> groups;
  std::vector<int32_t> tok, slot;  // per grouped row: x row, Y slot
  for (int e = 0; e < E + S; ++e) {
    Grp g{e, (int64_t)tok.size(), 0};
    for (int64_t t = 0; t < m; ++t) {
      if (e < E) {
        for (int k = 0; k < K; ++k)
          if (hids[t * K + k] == e) {
            tok.push_back((int32_t)t);
            slot.push_back((int32_t)(t * K + k));
          }
      } else {
        tok.push_back((int32_t)t);
        slot.push_back((int32_t)(m * K + (int64_t)(e - E) * m + t));
      }
    }
    g.rows = (int64_t)tok.size() - g.off;
    if (g.rows > 0) groups.push_back(g);
  }
  const int64_t R = (int64_t)tok.size();  // grouped rows
  const int64_t f_max = moe->f_max;
  // ---- workspace
  Arena ar;
  std::vector<size_t> o_img1(groups.size()), o_img2(groups.size());
  int64_t tiles_tot = 0;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const int nt = pf_ntok(groups[gi].rows);
    const int64_t tiles = (groups[gi].rows + nt - 1) / nt;
    tiles_tot += tiles;
    o_img1[gi] = ar.take((size_t)tiles * (d / kPfK) * nt * 128);
    o_img2[gi] = ar.take((size_t)tiles * (f_max / kPfK) * nt * 128);
  }
  const size_t o_h = ar.take((size_t)R * f_max * 2);
  const size_t o_y = ar.take((size_t)(m * K + (int64_t)S * m) * d * 4);
  // t problems: up to 3 per group
  std::vector<TProb> tps[2];
  std::vector<size_t> o_timg[3], o_part[3];
  for (int j = 0; j < 3; ++j) {
    o_timg[j].assign(groups.size(), 0);
    o_part[j].assign(groups.size(), 0);
  }
  for (size_t gi = 0; gi < groups.size(); ++gi)
    for (int j = 0; j < 3; ++j) {
      const milo_comp* c = moe->hc[groups[gi].e][j];
      if (!c || c->rank == 0) continue;
      const int64_t rows = groups[gi].rows;
      const int nt = pf_ntok(rows);
      const int64_t tiles = (rows + nt - 1) / nt;
      const int64_t kk = moe->hw[groups[gi].e][j]->rows;
      o_timg[j][gi] = ar.take((size_t)tiles * c->rch * 2 * nt * 128);
      o_part[j][gi] = ar.take(ImgTPlan::part_bytes(rows, kk, c, sms));
    }
  // every per-call table (token / slot lists, image, t and GEMM problem tables)
  // lives in one region, uploaded by one copy before the first kernel
  const size_t tab_bytes = 262144 + 2 * (((size_t)R * 4 + 255) & ~size_t(255));
  const size_t o_tab = ar.take(tab_bytes);
  void* mem = nullptr;
  {
    const milo_status ws_st = get_pf_ws(stream, ar.size, &mem);
    if (ws_st != MILO_OK) return ws_st;
  }
  uint8_t* base = static_cast<uint8_t*>(mem);
  __half* hbuf = reinterpret_cast<__half*>(base + o_h);
  float* Y = reinterpret_cast<float*>(base + o_y);
  uint8_t* tab = base + o_tab;
  milo_status st = MILO_OK;
  auto guard = [&](cudaError_t e) {
    if (e != cudaSuccess && st == MILO_OK) st = fail(MILO_ERR_CUDA, "prefill: %s", cudaGetErrorString(e));
  };
  hmark("planned+alloc");
  size_t tab_off = 0;
  auto upload = [&](const void* src, size_t bytes) -> uint8_t* {
    uint8_t* dst = tab + tab_off;
    tab_off = (tab_off + bytes + 255) & ~size_t(255);
    if (tab_off > tab_bytes) {
      if (st == MILO_OK) st = fail(MILO_ERR_CUDA, "prefill: table region overflow");
      return tab;
    }
    if (bytes && src) guard(h2d_async(dst, src, bytes, stream));
    return dst;
  };
  int32_t* dtok = nullptr;
  int32_t* dslot = nullptr;
  const int n_tprob[2] = {1, 1};  // k splits sized per problem (several CTAs per SM stay resident)
  // one grouped launch per phase: images (+ gathered rows) and the LoRC t partials
  auto img_t_phase = [&](int phase) {
    ImgTPlan plan;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      const int e = groups[gi].e;
      const int nt = pf_ntok(groups[gi].rows);
      const int mats[2] = {phase == 0 ? 0 : 2, phase == 0 ? 1 : 2};
      const milo_comp* cs[2] = {moe->hc[e][mats[0]], phase == 0 ? moe->hc[e][mats[1]] : nullptr};
      uint8_t* timg[2] = {base + o_timg[mats[0]][gi], base + o_timg[mats[1]][gi]};
      float* part[2] = {reinterpret_cast<float*>(base + o_part[mats[0]][gi]),
                        reinterpret_cast<float*>(base + o_part[mats[1]][gi])};
      if (phase == 0)
        plan.add(x, x_dtype, d, dtok + groups[gi].off, groups[gi].rows, d, nt, base + o_img1[gi], cs, timg, part, 2);
      else
        plan.add(hbuf + groups[gi].off * f_max, 1, f_max, nullptr, groups[gi].rows, moe->hw[e][2]->rows, nt,
                 base + o_img2[gi], cs, timg, part, 1);
    }
    guard(plan.launch_all(upload(nullptr, plan.table_bytes()), stream));
    std::vector<TProb> tv;
    int units = 0;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      const int e = groups[gi].e;
      const int nt = pf_ntok(groups[gi].rows);
      for (int mi : {phase == 0 ? 0 : 2, phase == 0 ? 1 : -1}) {
        if (mi < 0) continue;
        const milo_comp* c = moe->hc[e][mi];
        if (!c || c->rank == 0) continue;
        int u = 0;
        if (phase == 0)
          tv.push_back(make_tprob(x, x_dtype, d, dtok + groups[gi].off, groups[gi].rows, d, nt, c,
                                  base + o_timg[mi][gi], reinterpret_cast<float*>(base + o_part[mi][gi]), sms, units, &u,
                                  n_tprob[phase]));
        else
          tv.push_back(make_tprob(hbuf + groups[gi].off * f_max, 1, f_max, nullptr, groups[gi].rows,
                                  moe->hw[e][2]->rows, nt, c, base + o_timg[mi][gi],
                                  reinterpret_cast<float*>(base + o_part[mi][gi]), sms, units, &u, n_tprob[phase]));
        units += u;
      }
    }
    guard(launch_t_batch(tv, units, upload(nullptr, tv.size() * sizeof(TProb)), stream));
  };
  auto sequence = [&] {
    tab_off = 0;
    dtok = reinterpret_cast<int32_t*>(upload(tok.data(), (size_t)R * 4));
    dslot = reinterpret_cast<int32_t*>(upload(slot.data(), (size_t)R * 4));
    // ---- phase 1: x rows -> images, t1, t3; w1|w3 + LoRC + SwiGLU -> h
    img_t_phase(0);
    hmark(g_dry ? "dry: phase1 imgs" : "phase1 imgs launched");
    {
      std::vector<PfProblem> pv;
      for (size_t gi = 0; gi < groups.size(); ++gi) {
        const int e = groups[gi].e;
        PfProblem P{};
        P.w[0] = moe->hw[e][0]->tiles;
        P.w[1] = moe->hw[e][1]->tiles;
        P.act = base + o_img1[gi];
        for (int mi = 0; mi < 2; ++mi) {
          const milo_comp* c = moe->hc[e][mi];
          if (c && c->rank > 0) {
            P.vimg[mi] = c->vimg;
            P.timg[mi] = base + o_timg[mi][gi];
            P.rchunks[mi] = c->rch;
          }
        }
        P.k = (int32_t)d;
        P.n = (int32_t)moe->hw[e][0]->cols;
        P.rows = (int32_t)groups[gi].rows;
        P.ntok = pf_ntok(groups[gi].rows);
        P.mode = moe->hw[e][0]->mode;
        P.kind = 1;
        P.out_dtype = 1;
        P.ldo = f_max;
        P.out = hbuf + groups[gi].off * f_max;
        pv.push_back(P);
      }
      if (st == MILO_OK)
        st = launch_prefill<2>(pv.data(), (int)pv.size(), stream, sms,
                               upload(nullptr, pv.size() * sizeof(PfProblem) + 4096));
    }
    (void)tiles_tot;
    // ---- phase 2: h rows -> images, t2; w2 + LoRC -> Y slots
    hmark(g_dry ? "dry: gemm1" : "gemm1 launched");
    if (st == MILO_OK) img_t_phase(1);
    hmark(g_dry ? "dry: phase2 imgs" : "phase2 imgs launched");
    if (st == MILO_OK) {
      std::vector<PfProblem> pv;
      for (size_t gi = 0; gi < groups.size(); ++gi) {
        const int e = groups[gi].e;
        PfProblem P{};
        P.w[0] = moe->hw[e][2]->tiles;
        P.act = base + o_img2[gi];
        const milo_comp* c = moe->hc[e][2];
        if (c && c->rank > 0) {
          P.vimg[0] = c->vimg;
          P.timg[0] = base + o_timg[2][gi];
          P.rchunks[0] = c->rch;
        }
        P.k = (int32_t)moe->hw[e][2]->rows;
        P.n = (int32_t)d;
        P.rows = (int32_t)groups[gi].rows;
        P.ntok = pf_ntok(groups[gi].rows);
        P.mode = moe->hw[e][2]->mode;
        P.kind = 0;
        P.out_dtype = 0;
        P.ldo = d;
        P.out = Y;
        P.row_map = dslot + groups[gi].off;
        pv.push_back(P);
      }
      st = launch_prefill<1>(pv.data(), (int)pv.size(), stream, sms,
                             upload(nullptr, pv.size() * sizeof(PfProblem) + 4096));
    }
    if (st == MILO_OK) {
      const int64_t total = m * (d / 4);
      const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
      guard(launch(moe_combine_kernel, dim3(grid), dim3(256), 0, stream, false, (const float*)Y,
                   (const int32_t*)ids, (const float*)wts, m, K, S, d, out, out_dtype));
    }
  };
  // pass 1 records the uploads (no launches), one coalesced copy, pass 2 launches
  struct PassReset {  // leave the thread's staging state clean on every exit
    ~PassReset() {
      g_dry = false;
      g_pin.mode = 0;
      g_pin.rec.clear();
      g_pin.lo = g_pin.hi = nullptr;
    }
  } pass_reset;
  pin_begin();
  g_pin.lo = tab;
  g_pin.hi = tab + tab_bytes;
  g_pin.mode = 1;
  g_dry = true;
  sequence();
  g_dry = false;
  g_pin.mode = 0;
  if (st == MILO_OK) guard(pin_flush(stream));
  hmark("uploads issued");
  if (st == MILO_OK) {
    g_pin.mode = 2;
    sequence();
    g_pin.mode = 0;
  }
  pin_end(stream);
  return st;
}

// The MoE prefill path with the plan on the device (moe_plan_kernel): router ->
// plan -> per phase: activation images, LoRC t, the tcgen05 grouped GEMM ->
// combine, all stream-ordered (no host synchronisation, graph-capturable).
// Workspace regions are sized here for the worst routing of m tokens; the
// launches use host grid bounds and read their sizes from the plan.
milo_status moe_prefill_dev(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype, const float* logits,
                            int32_t* ids, float* wts, void* out, int32_t out_dtype, cudaStream_t stream, int sms) {
  const int E = moe->E, K = moe->K, S = moe->n_shared;
  const int64_t d = moe->d, f_max = moe->f_max;
  const int64_t G = E + S, R = m * K + (int64_t)S * m;
  if (G > kPlanMaxGroups) return fail(MILO_ERR_CONFIG, "prefill: more than %d experts", kPlanMaxGroups);
  if (K > 0 && logits)
    CUDA_TRY(launch(router_topk_kernel, dim3((unsigned)((m + 7) / 8)), dim3(256), 0, stream, false, logits, m, E, K,
                    moe->score_mode, ids, wts));
  // ---- worst-case regions (tiles x ntok <= rows + 127 per group)
  const int64_t rows_b = R + 127 * G;
  int64_t kmax[3] = {d, d, 0};
  for (int i = 0; i < (int)G; ++i) kmax[2] = std::max<int64_t>(kmax[2], (int64_t)moe->hw[i][2]->rows);
  Arena ar;
  const size_t o_img0 = ar.take((size_t)rows_b * d * 2 + 256 * G);
  const size_t o_img1 = ar.take((size_t)rows_b * f_max * 2 + 256 * G);
  size_t o_timg[3], o_part[3];
  for (int j = 0; j < 3; ++j) {
    o_timg[j] = ar.take((size_t)rows_b * moe->rch_max[j] * 256 + 256 * G);
    o_part[j] = ar.take((size_t)(kmax[j] / kPfK) * R * moe->rch_max[j] * 256 + 256 * G);
  }
  const size_t o_h = ar.take((size_t)R * f_max * 2);
  const size_t o_y = ar.take((size_t)R * d * 4);
  const size_t o_tok = ar.take((size_t)R * 4);
  const size_t o_slot = ar.take((size_t)R * 4);
  size_t o_jobs[2], o_tps[2], o_probs[2], o_starts[2];
  for (int ph = 0; ph < 2; ++ph) {
    o_jobs[ph] = ar.take((size_t)G * sizeof(ImgJob));
    o_tps[ph] = ar.take((size_t)G * (ph == 0 ? 2 : 1) * sizeof(TProb));
    o_probs[ph] = ar.take((size_t)G * sizeof(PfProblem));
    o_starts[ph] = ar.take((size_t)(G + 1) * 4);
  }
  const size_t o_counts = ar.take(32 * 4);
  void* mem = nullptr;
  {
    const milo_status ws_st = get_pf_ws(stream, ar.size, &mem);
    if (ws_st != MILO_OK) return ws_st;
  }
  uint8_t* b = static_cast<uint8_t*>(mem);
  PfPlanArgs pa{};
  pa.ids = ids;
  pa.m = m;
  pa.K = K;
  pa.E = E;
  pa.S = S;
  pa.sms = sms;
  pa.ex = moe->pf_static;
  pa.x = x;
  pa.x_dtype = x_dtype;
  pa.d = d;
  pa.f_max = f_max;
  pa.tok = reinterpret_cast<int32_t*>(b + o_tok);
  pa.slot = reinterpret_cast<int32_t*>(b + o_slot);
  for (int ph = 0; ph < 2; ++ph) {
    pa.jobs[ph] = reinterpret_cast<ImgJob*>(b + o_jobs[ph]);
    pa.tps[ph] = reinterpret_cast<TProb*>(b + o_tps[ph]);
    pa.probs[ph] = reinterpret_cast<PfProblem*>(b + o_probs[ph]);
    pa.starts[ph] = reinterpret_cast<int32_t*>(b + o_starts[ph]);
  }
  pa.counts = reinterpret_cast<int32_t*>(b + o_counts);
  pa.img[0] = b + o_img0;
  pa.img[1] = b + o_img1;
  for (int j = 0; j < 3; ++j) {
    pa.timg[j] = b + o_timg[j];
    pa.part[j] = b + o_part[j];
  }
  pa.h = reinterpret_cast<__half*>(b + o_h);
  pa.Y = reinterpret_cast<float*>(b + o_y);
  // (programmatic launches of this chain measured no faster: the early CTAs of
  // each dependent grid hold SM slots while the previous grid drains)
  pa.dbg = g_dbg ? g_dbg + 2 * kPfDbgLongs : nullptr;  // after the two GEMM phases' regions
  // w2 items of two n-tiles (one activation image feeds two MMAs; half the items)
  static const int ng2_env = [] {
    const char* e = getenv("MILO_PF_NG2");
    return e ? atoi(e) : 1;
  }();
  pa.ng2 = (ng2_env && d % (2 * kPfM) == 0) ? 1 : 0;
  // cached ids + the per-warp expert histograms of the window scans
  const size_t ids_smem = (((size_t)m * K + 3) & ~size_t(3)) * 4 + (size_t)32 * kPlanMaxGroups * 4;
  pa.ids_cached = ids_smem <= kPlanIdsSmem ? 1 : 0;
  {
    static thread_local int plan_dev = -1;
    int dv = 0;
    cudaGetDevice(&dv);
    if (plan_dev != dv) {
      CUDA_TRY(cudaFuncSetAttribute(moe_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPlanIdsSmem));
      plan_dev = dv;
    }
  }
  CUDA_TRY(launch(moe_plan_kernel, dim3(1), dim3(1024), pa.ids_cached ? ids_smem : 0, stream, false, pa));
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    CUDA_TRY(cudaFuncSetAttribute(pf_img_t_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kImgTSmem));
    CUDA_TRY(set_smem(pf_gemm_kernel<2, 1>, PfCfg<2, 1>::kBytes));
    CUDA_TRY(set_smem(pf_gemm_kernel<1, 1>, PfCfg<1, 1>::kBytes));
    CUDA_TRY(set_smem(pf_gemm_kernel<1, 2>, PfCfg<1, 2>::kBytes));
    configured_dev = dev;
  }
  for (int ph = 0; ph < 2; ++ph) {
    const int32_t* cnt = pa.counts + 16 * ph;
    // activation images (+ gathered rows) and LoRC t = x U -> hi / lo images
    CUDA_TRY(launch(pf_img_t_kernel<false>, dim3((unsigned)(sms * 8)), dim3(256), 0, stream, false,
                    (const ImgJob*)pa.jobs[ph], 0, cnt));
    if (moe->t_kinds[ph] & 1)
      CUDA_TRY(launch(pf_t_kernel<0>, dim3((unsigned)(sms * 8)), dim3(256), 0, stream, false, (const TProb*)pa.tps[ph],
                      0, cnt + 2));
    if (moe->t_kinds[ph] & 2)
      CUDA_TRY(launch(pf_t_kernel<1>, dim3((unsigned)(sms * 8)), dim3(256), 0, stream, false, (const TProb*)pa.tps[ph],
                      0, cnt + 2));
    CUDA_TRY(launch(pf_t_images_kernel, dim3(64, (unsigned)std::max<int64_t>(1, G * (ph == 0 ? 2 : 1))), dim3(256),
                    0, stream, false, (const TProb*)pa.tps[ph], 0, cnt + 2));
    // the grouped tcgen05 GEMM (persistent grid; items from the plan)
    PfArgs a{};
    a.dbg = g_dbg ? g_dbg + ph * kPfDbgLongs : nullptr;  // one timeline region per phase
    a.flags = g_dbg_flags;
    a.problems = pa.probs[ph];
    a.item_start = pa.starts[ph];
    a.dev_counts = cnt + 4;
    a.ntok_max = kPfN;
    a.n_items = 1;
    if (ph == 0) {
      ProfScope ps(kProfGemv1, stream);
      CUDA_TRY(launch(pf_gemm_kernel<2, 1>, dim3(sms), dim3(PfRoles<2, 1>::kThreads), PfCfg<2, 1>::kBytes, stream,
                      false, a));
    } else {
      ProfScope ps(kProfGemv2, stream);
      if (pa.ng2)
        CUDA_TRY(launch(pf_gemm_kernel<1, 2>, dim3(sms), dim3(PfRoles<1, 2>::kThreads), PfCfg<1, 2>::kBytes, stream,
                        false, a));
      else
        CUDA_TRY(launch(pf_gemm_kernel<1, 1>, dim3(sms), dim3(PfRoles<1, 1>::kThreads), PfCfg<1, 1>::kBytes, stream,
                        false, a));
    }
  }
  const int64_t total = m * (d / 4);
  const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
  CUDA_TRY(launch(moe_combine_kernel, dim3(grid), dim3(256), 0, stream, false, (const float*)pa.Y,
                  (const int32_t*)ids, (const float*)wts, m, K, S, d, out, out_dtype));
  return MILO_OK;
}

// logits != nullptr: the route kernel computes the top-k into ids / wts
// (outputs); otherwise ids / wts are the given routing (inputs).
// ---------------------------------------------------------------------------
// hdec_kernel (hdec.cuh): the decode-regime layer, h-local.  Workspace: the
// tagged regions (T partials, P1 partials, published h) in the decode data
// region (0xFF-filled when allocated, so no stale tag matches), the fp32
// accumulators (zeroed by the kernel itself) and a two-parity control block
// (each call zeroes the block the next call on this workspace uses).
// ---------------------------------------------------------------------------
int hdec_env() {
  static const int v = [] {
    const char* e = getenv("MILO_HDEC");
    return e ? atoi(e) : 0;  // opt-in until it beats the round-1 megakernel everywhere
  }();
  return v;
}

bool hdec_eligible(const milo_moe* moe, int64_t m) {
  if (hdec_env() == 0 || legacy_path() || !moe->hd_ok || m < 1 || m > kHdMaxTok) return false;
  const int64_t np_max = std::min<int64_t>(moe->E, m * moe->K) + moe->n_shared;
  return np_max <= kHdMaxParts && moe->E <= 256 && moe->K <= 16 && moe->d % 64 == 0 && moe->d >= 64;
}

template <int NT>
milo_status launch_hdec(const milo_moe* moe, const void* x, int64_t m, int32_t x_dtype, const float* logits,
                        int32_t* ids, float* wts, void* out, int32_t out_dtype, cudaStream_t stream, int sms) {
  using CF = HdCfg<NT>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (configured_dev != dev) {
    CUDA_TRY(set_smem(hdec_kernel<NT>, CF::kBytes));
    configured_dev = dev;
  }
  const int G = sms * CF::kCtasPerSm;
  const int64_t KT = moe->d / 32, nch = (KT + kHdTK - 1) / kHdTK;
  const int64_t np_max = std::min<int64_t>(moe->E, m * moe->K) + moe->n_shared;
  const int64_t r16 = std::max(moe->r16_max, 16);
  Arena ar;
  const size_t o_tp = ar.take((size_t)np_max * 2 * (r16 / 16) * nch * 16 * 16 * 8);
  const size_t o_pt = ar.take((size_t)G * 1024 * NT * 8);
  const size_t o_hp = ar.take((size_t)G * 16 * 32 * 8);
  const size_t o_t2 = ar.take((size_t)(m * moe->K + moe->n_shared * m) * r16 * 4);
  const size_t o_ac = ar.take(out_dtype == 0 ? 0 : (size_t)m * moe->d * 4);
  const size_t o_x = ar.take(x_dtype == 0 ? (size_t)m * moe->d * 2 : 0);
  DecodeWs* w = nullptr;
  int epoch = 0;
  milo_status st = get_ws(stream, ar.size, &w, &epoch);
  if (st != MILO_OK) return st;
  uint32_t parity = 0;
  {
    std::lock_guard<std::mutex> lock(g_ws_mu);
    if (!w->hctrl) {
      CUDA_TRY(cudaMalloc(&w->hctrl, 2 * kHdCtrl * 4));
      CUDA_TRY(cudaMemsetAsync(w->hctrl, 0, 2 * kHdCtrl * 4, stream));
      w->hcalls = 0;
    }
    parity = w->hcalls++ & 1u;
  }
  uint8_t* base = static_cast<uint8_t*>(w->data);
  HdArgs a{};
  a.m = (int32_t)m;
  a.E = moe->E;
  a.K = moe->K;
  a.S = moe->n_shared;
  a.score_mode = moe->score_mode;
  a.d = moe->d;
  a.logits = logits;
  a.ids_in = logits ? nullptr : ids;
  a.wts_in = logits ? nullptr : wts;
  a.ids_out = logits ? ids : nullptr;
  a.wts_out = logits ? wts : nullptr;
  a.experts = moe->dec_experts;
  a.hexp = moe->hd_exp;
  a.w2maps = moe->hd_w2maps;
  a.x = static_cast<const __half*>(x);
  a.ldx = moe->d;
  if (x_dtype == 0) {  // the kernel streams binary16 rows: round f32 rows once (gemm.cpp:144-146)
    __half* x16 = reinterpret_cast<__half*>(base + o_x);
    const int64_t n4 = m * (moe->d / 4);
    const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)sms * 4);
    CUDA_TRY(launch(rows_to_half_kernel, dim3(std::max(grid, 1)), dim3(256), 0, stream, false,
                    static_cast<const float*>(x), m, (int64_t)moe->d, (int64_t)moe->d, x16));
    a.x = x16;
  }
  a.out = out;
  a.out_dtype = out_dtype;
  a.ldo = moe->d;
  a.epoch = epoch;
  a.ctrl = w->hctrl + parity * kHdCtrl;
  a.ctrl_next = w->hctrl + (parity ^ 1u) * kHdCtrl;
  a.tpart = reinterpret_cast<uint64_t*>(base + o_tp);
  a.part = reinterpret_cast<uint64_t*>(base + o_pt);
  a.hpub = reinterpret_cast<uint64_t*>(base + o_hp);
  a.t2acc = reinterpret_cast<float*>(base + o_t2);
  a.acc = out_dtype == 0 ? nullptr : reinterpret_cast<float*>(base + o_ac);
  a.dbg = g_dbg;
  a.dbg_flags = g_dbg_flags;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(CF::kThreads);
  cfg.dynamicSmemBytes = CF::kBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (g_dry) return MILO_OK;
  ++g_launches;
  ProfScope ps(kProfGemv1, stream);
  CUDA_TRY(cudaLaunchKernelEx(&cfg, hdec_kernel<NT>, a));
  return MILO_OK;
}

milo_status moe_forward_impl(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype,
                             const float* logits, int32_t* ids, float* wts, void* out,
                             int32_t out_dtype, void* stream_) {
  if (!moe) return fail(MILO_ERR_ARGUMENT, "null moe");
  if (m < 0) return fail(MILO_ERR_SHAPE, "negative token count");
  if (m == 0) return MILO_OK;
  if (!x || !out || (moe->K > 0 && (!ids || !wts))) return fail(MILO_ERR_ARGUMENT, "null argument");
  if ((x_dtype != 0 && x_dtype != 1) || (out_dtype != 0 && out_dtype != 1))
    return fail(MILO_ERR_ARGUMENT, "unsupported dtype");
  DeviceProps props = device_props();
  if (!props.ok || props.major != 10) return fail(MILO_ERR_CUDA, "no sm_100 device");
  cudaStream_t stream = (cudaStream_t)stream_;
  if (hdec_eligible(moe, m))
    return m <= 8 ? launch_hdec<1>(moe, x, m, x_dtype, logits, ids, wts, out, out_dtype, stream, props.sms)
                  : launch_hdec<2>(moe, x, m, x_dtype, logits, ids, wts, out, out_dtype, stream, props.sms);
  // decode megakernel blocks: each touched expert's tokens in chunks of m_pad rows
  // 8-row blocks (NT = 1) up to batch 24: an expert with more tokens takes two
  // blocks (its weights stream twice) but the 16-row variant's MMA work and
  // spills cost more (Mixtral batch 16: 332 -> 285 us; MILO_DEC_NT1_MAX overrides)
  static const int nt1_max = [] {
    const char* e = getenv("MILO_DEC_NT1_MAX");
    return e ? atoi(e) : 24;
  }();
  const int dec_mpad = m <= nt1_max ? 8 : 16;
  // bound on the blocks: t = min(E, mK) touched experts, an expert with c <= m
  // entries needs ceil(c / m_pad) blocks (one each when m <= m_pad), so at most
  // t + (mK - t) / m_pad, plus the shared experts' chunks
  const int64_t n_ent = m * moe->K, t_max = std::min<int64_t>(moe->E, n_ent);
  const int64_t nb_dec = t_max + (m <= dec_mpad ? 0 : (n_ent - t_max) / dec_mpad) +
                         (int64_t)moe->n_shared * ((m + dec_mpad - 1) / dec_mpad);
  static const int dec_max_m = [] {  // experiments: MILO_DEC_MAX_M caps the decode megakernel's batch
    const char* e = getenv("MILO_DEC_MAX_M");
    return e ? std::min(atoi(e), kDecMaxM) : kDecMaxM;
  }();
  if (!legacy_path() && m <= dec_max_m && m * moe->K <= kDecMaxEntries && nb_dec <= kDecMaxBlocks &&
      moe->E <= 256 && moe->K <= 16 && moe->d / 64 <= 4096) {
    DecArgs a{};
    a.moe = 1;
    a.m = (int32_t)m;
    a.logits = logits;
    a.ids_in = logits ? nullptr : ids;
    a.wts_in = logits ? nullptr : wts;
    a.ids_out = logits ? ids : nullptr;
    a.wts_out = logits ? wts : nullptr;
    a.E = moe->E;
    a.K = moe->K;
    a.S = moe->n_shared;
    a.score_mode = moe->score_mode;
    a.experts = moe->dec_experts;
    a.d = moe->d;
    a.out = out;
    a.out_dtype = out_dtype;
    a.ldo = moe->d;
    const int64_t y_rows = m * moe->K + (int64_t)moe->n_shared * m;
    return m <= nt1_max ? launch_decode<1, 2, true>(a, x, x_dtype, moe->d, (int)nb_dec, moe->f_max,
                                              moe->r16_max, y_rows, stream, props.sms)
                  : launch_decode<2, 2, true>(a, x, x_dtype, moe->d, (int)nb_dec, moe->f_max,
                                              moe->r16_max, y_rows, stream, props.sms);
  }
  if (!legacy_path() && moe->prefill_ok && m > kDecMaxTok && m >= prefill_min_rows() / 2 &&
      (int64_t)m * std::max(1, moe->K) + (int64_t)moe->n_shared * m < (1 << 30))
  {
    static const bool host_plan = getenv("MILO_PF_HOSTPLAN") != nullptr;  // A/B: the round-1 host planner
    return host_plan ? moe_prefill(moe, x, m, x_dtype, logits, ids, wts, out, out_dtype, stream, props.sms)
                     : moe_prefill_dev(moe, x, m, x_dtype, logits, ids, wts, out, out_dtype, stream, props.sms);
  }
  // Shapes the prefill kernel cannot take (e.g. f % 128 == 64) beyond the decode
  // megakernel's batch: independent token chunks, each one decode-megakernel call.
  if (!legacy_path() && m > dec_max_m && moe->E <= 256 && moe->K <= 16 && moe->d / 64 <= 4096) {
    int64_t c = dec_max_m;
    auto fits = [&](int64_t cm) {
      const int64_t ne = cm * moe->K, tm = std::min<int64_t>(moe->E, ne), mp = cm <= 8 ? 8 : 16;
      const int64_t nb = tm + (cm <= mp ? 0 : (ne - tm) / mp) + (int64_t)moe->n_shared * ((cm + mp - 1) / mp);
      return ne <= kDecMaxEntries && nb <= kDecMaxBlocks;
    };
    while (c > 1 && !fits(c)) c /= 2;
    if (fits(c)) {
      const size_t xs = x_dtype == 0 ? 4 : 2, os = out_dtype == 0 ? 4 : 2;
      for (int64_t t0 = 0; t0 < m; t0 += c) {
        const int64_t mm = std::min(c, m - t0);
        const milo_status st = moe_forward_impl(
            moe, static_cast<const uint8_t*>(x) + t0 * moe->d * xs, mm, x_dtype, logits ? logits + t0 * moe->E : nullptr,
            ids ? ids + t0 * moe->K : nullptr, wts ? wts + t0 * moe->K : nullptr,
            static_cast<uint8_t*>(out) + t0 * moe->d * os, out_dtype, stream_);
        if (st != MILO_OK) return st;
      }
      return MILO_OK;
    }
  }
  // The round-1 multi-launch path: only with MILO_LEGACY=1 (A/B) or shapes outside every
  // kernel's limits.  Token chunks keep every launch under the problem-table bound.
  const int nt = m <= 8 ? 1 : 2;
  const int m_pad = 8 * nt;
  const int64_t per_tok = std::max(1, moe->K) + moe->n_shared;
  const int64_t chunk = std::max<int64_t>(
      m_pad, ((int64_t)(kMaxProblems - 1 - moe->E - moe->n_shared) * m_pad) / per_tok / m_pad * m_pad);
  for (int64_t t0 = 0; t0 < m; t0 += chunk) {
    const int64_t mm = std::min(chunk, m - t0);
    const size_t xs = x_dtype == 0 ? 4 : 2, os = out_dtype == 0 ? 4 : 2;
    const void* xc = static_cast<const uint8_t*>(x) + t0 * moe->d * xs;
    void* oc = static_cast<uint8_t*>(out) + t0 * moe->d * os;
    int32_t* ic = ids ? ids + t0 * moe->K : nullptr;
    float* wc = wts ? wts + t0 * moe->K : nullptr;
    const float* lc = logits ? logits + t0 * moe->E : nullptr;
    milo_status st =
        nt == 1 ? moe_run<1>(moe, xc, mm, x_dtype, lc, ic, wc, oc, out_dtype, stream, props.sms)
                : moe_run<2>(moe, xc, mm, x_dtype, lc, ic, wc, oc, out_dtype, stream, props.sms);
    if (st != MILO_OK) return st;
  }
  return MILO_OK;
}

}  // namespace

extern "C" milo_status milo_moe_forward_routed(milo_moe* moe, const void* x, int64_t m,
                                               int32_t x_dtype, const int32_t* ids,
                                               const float* wts, void* out, int32_t out_dtype,
                                               void* stream) {
  return moe_forward_impl(moe, x, m, x_dtype, nullptr, const_cast<int32_t*>(ids),
                          const_cast<float*>(wts), out, out_dtype, stream);
}

extern "C" milo_status milo_moe_forward(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype,
                                        const float* logits, void* out, int32_t out_dtype,
                                        int32_t* topk_ids, float* topk_w, void* stream_) {
  if (!moe) return fail(MILO_ERR_ARGUMENT, "null moe");
  if (m <= 0) return m == 0 ? MILO_OK : fail(MILO_ERR_SHAPE, "negative token count");
  if (moe->K > 0 && !logits) return fail(MILO_ERR_ARGUMENT, "null router logits");
  cudaStream_t stream = (cudaStream_t)stream_;
  int32_t* ids = topk_ids;
  float* w = topk_w;
  void* mem = nullptr;
  if (moe->K > 0 && (!ids || !w)) {
    CUDA_TRY(cudaMallocAsync(&mem, (size_t)m * moe->K * 8, stream));
    ids = static_cast<int32_t*>(mem);
    w = reinterpret_cast<float*>(ids + m * moe->K);
  }
  milo_status st = moe_forward_impl(moe, x, m, x_dtype, moe->K > 0 ? logits : nullptr, ids, w,
                                    out, out_dtype, stream);
  if (mem) cudaFreeAsync(mem, stream);
  return st;
}

// Expert-parallel exchange helpers (include/milo_b200.h).
extern "C" milo_status milo_ep_dispatch(const int32_t* ids, int64_t m, int32_t K, int32_t world,
                                        int32_t per, int32_t capacity, const void* x, int32_t x_dtype,
                                        int64_t d, void* send_x, int64_t ld_send, int32_t* send_meta,
                                        int32_t* slot, void* stream) {
  if (m < 0 || K < 1 || world < 1 || per < 1 || capacity < m * K || m * K > 1024 ||
      (int64_t)world * capacity > 8192 || d % 8 != 0)
    return fail(MILO_ERR_CONFIG, "ep_dispatch: unsupported sizes (m K <= 1024, world x capacity <= 8192)");
  if (ld_send % 8 != 0 || ld_send < (send_meta ? d : d + 8))
    return fail(MILO_ERR_CONFIG, "ep_dispatch: row stride must be a multiple of 8 and hold the id columns");
  if (m == 0) return MILO_OK;
  CUDA_TRY(launch(ep_dispatch_kernel, dim3(1), dim3(1024), 0, (cudaStream_t)stream, false, ids,
                  (int32_t)(m * K), K, world, per, capacity, x, x_dtype, d, static_cast<__half*>(send_x), ld_send,
                  send_meta, slot));
  return MILO_OK;
}

extern "C" milo_status milo_ep_combine(const float* y, const int32_t* slot, const float* wts, int64_t m,
                                       int32_t K, int64_t d, float* out, void* stream) {
  if (m <= 0) return m == 0 ? MILO_OK : fail(MILO_ERR_SHAPE, "negative token count");
  if (d % 4 != 0) return fail(MILO_ERR_SHAPE, "d must be a multiple of 4");
  const int64_t total = m * (d / 4);
  CUDA_TRY(launch(ep_combine_kernel, dim3((unsigned)std::min<int64_t>((total + 255) / 256, 1184)), dim3(256), 0,
                  (cudaStream_t)stream, false, y, slot, wts, m, K, d, out, (const float*)nullptr));
  return MILO_OK;
}

constexpr size_t kHostZeroCopyMax = 256 * 1024;  // output bytes written over the host link directly

extern "C" milo_status milo_router_gemm(const void* x, int64_t m, int64_t d, int32_t x_dtype, const uint16_t* gate,
                                        int32_t E, float* logits, void* stream) {
  if (m < 0 || d < 1 || E < 1) return fail(MILO_ERR_SHAPE, "router gemm: bad shape");
  if (x_dtype != MILO_F32 && x_dtype != MILO_F16) return fail(MILO_ERR_ARGUMENT, "router gemm: x dtype");
  if (m == 0) return MILO_OK;
  if (!x || !gate || !logits) return fail(MILO_ERR_ARGUMENT, "null argument");
  const int warps = 8;
  const int64_t outs = m * E;
  CUDA_TRY(launch(router_gemm_kernel, dim3((unsigned)((outs + warps - 1) / warps)), dim3(32 * warps), 0,
                  (cudaStream_t)stream, true, x, x_dtype, d, m, d, reinterpret_cast<const __half*>(gate), E, logits));
  return MILO_OK;
}

extern "C" milo_status milo_moe_set_gate(milo_moe* moe, const uint16_t* gate, int64_t E, int64_t d) {
  if (!moe || !gate) return fail(MILO_ERR_ARGUMENT, "null argument");
  if (E != moe->E || d != moe->d)
    return fail(MILO_ERR_SHAPE, "gate is %lld x %lld, the layer needs %d x %d", (long long)E, (long long)d, moe->E,
                moe->d);
  void* g = nullptr;
  CUDA_TRY(cudaMalloc(&g, (size_t)E * d * 2));
  const cudaError_t e = cudaMemcpy(g, gate, (size_t)E * d * 2, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(g);
    return fail(MILO_ERR_CUDA, "%s", cudaGetErrorString(e));
  }
  if (moe->gate) cudaFree(moe->gate);
  moe->gate = static_cast<__half*>(g);
  return MILO_OK;
}

extern "C" milo_status milo_moe_forward_x(milo_moe* moe, const void* x, int64_t m, int32_t x_dtype, void* out,
                                          int32_t out_dtype, int32_t* topk_ids, float* topk_w, void* stream_) {
  if (!moe) return fail(MILO_ERR_ARGUMENT, "null moe");
  if (!moe->gate || moe->E == 0) return fail(MILO_ERR_CONFIG, "no router gate attached (milo_moe_set_gate)");
  if (m < 0) return fail(MILO_ERR_SHAPE, "negative token count");
  if (m == 0) return MILO_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  float* logits = nullptr;  // per-call, stream-ordered
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&logits), (size_t)m * moe->E * 4, stream));
  milo_status st = milo_router_gemm(x, m, moe->d, x_dtype, reinterpret_cast<const uint16_t*>(moe->gate), moe->E,
                                    logits, stream);
  if (st == MILO_OK) st = milo_moe_forward(moe, x, m, x_dtype, logits, out, out_dtype, topk_ids, topk_w, stream);
  const cudaError_t e = cudaFreeAsync(logits, stream);
  if (st == MILO_OK && e != cudaSuccess) st = fail(MILO_ERR_CUDA, "%s", cudaGetErrorString(e));
  return st;
}

extern "C" milo_status milo_moe_forward_host(milo_moe* moe, const float* x, int64_t m, int64_t x_cols,
                                             const float* logits, int64_t logit_cols, float* out) {
  if (!moe) return fail(MILO_ERR_ARGUMENT, "null moe");
  if (m < 0) return fail(MILO_ERR_SHAPE, "negative token count");
  // the reference's shape check order (gemm.cpp:135-136): activation columns first
  if (x_cols != moe->d) return fail(MILO_ERR_SHAPE, "x has %lld columns, the layer's d is %d", (long long)x_cols, moe->d);
  if (logit_cols != moe->E)
    return fail(MILO_ERR_SHAPE, "router logits have %lld columns, the layer has %d experts", (long long)logit_cols, moe->E);
  if (m == 0) return MILO_OK;
  if (!x || !out || (moe->E > 0 && !logits)) return fail(MILO_ERR_ARGUMENT, "null argument");
  cudaStream_t stream = nullptr;
  std::lock_guard<std::mutex> lock(moe->stage_mu);
  // x and logits go up in ONE copy from a pinned staging buffer (host memcpy is
  // cheaper than a second DMA launch at decode sizes); out comes back in one.
  const size_t xb = (size_t)m * moe->d * 4, lb = (size_t)m * std::max(moe->E, 0) * 4;
  const size_t lb16 = (lb + 15) & ~size_t(15);
  const size_t need = xb + lb16 + xb;
  if (moe->stage_bytes < need) {
    if (moe->host_stage) cudaFreeHost(moe->host_stage);
    if (moe->dev_stage) cudaFree(moe->dev_stage);
    moe->host_stage = moe->dev_stage = nullptr;
    moe->stage_bytes = 0;
    CUDA_TRY(cudaMallocHost(&moe->host_stage, need));
    CUDA_TRY(cudaMalloc(&moe->dev_stage, need));
    moe->stage_bytes = need;
  }
  uint8_t* hs = static_cast<uint8_t*>(moe->host_stage);
  uint8_t* b = static_cast<uint8_t*>(moe->dev_stage);
  // The h-local decode kernel streams binary16 rows and accumulates the output
  // with device-memory reductions: x is rounded to binary16 here (RNE, the
  // reference's half(A), gemm.cpp:144-146) and goes up at half the bytes; the
  // output comes back by one copy.
  const bool hd = hdec_eligible(moe, m);
  const size_t xup = hd ? (size_t)m * moe->d * 2 : xb;
  if (hd) {
    uint16_t* x16 = reinterpret_cast<uint16_t*>(hs);
    for (int64_t i = 0; i < m * (int64_t)moe->d; ++i) x16[i] = f32_to_f16_rne(x[i]);
  } else {
    std::memcpy(hs, x, xb);
  }
  if (lb) std::memcpy(hs + xup, logits, lb);
  cudaError_t e = cudaMemcpyAsync(b, hs, xup + lb, cudaMemcpyHostToDevice, stream);
  milo_status st = e == cudaSuccess ? MILO_OK : fail(MILO_ERR_CUDA, "%s", cudaGetErrorString(e));
  // Otherwise decode-sized outputs are written by the kernel straight into the
  // mapped pinned stage (posted writes over the host link, visible once the
  // stream has synchronised): no device-to-host copy on the critical path.
  void* out_dev = b + xb + lb16;
  const bool zero_copy = !hd && xb <= kHostZeroCopyMax &&
                         cudaHostGetDevicePointer(&out_dev, hs + xb + lb16, 0) == cudaSuccess;
  if (!zero_copy) {
    cudaGetLastError();
    out_dev = b + xb + lb16;
  }
  if (st == MILO_OK)
    st = milo_moe_forward(moe, b, m, hd ? MILO_F16 : MILO_F32, reinterpret_cast<float*>(b + xup), out_dev, MILO_F32,
                          nullptr, nullptr, stream);
  if (st == MILO_OK && !zero_copy) {
    e = cudaMemcpyAsync(hs + xb + lb16, b + xb + lb16, xb, cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) st = fail(MILO_ERR_CUDA, "%s", cudaGetErrorString(e));
  }
  e = cudaStreamSynchronize(stream);
  if (st == MILO_OK && e != cudaSuccess) st = fail(MILO_ERR_CUDA, "%s", cudaGetErrorString(e));
  if (st == MILO_OK) std::memcpy(out, hs + xb + lb16, xb);
  return st;
}

// ===========================================================================
// MILO1 container loaders.  Format of the
// reference's tensor store (tensor_store.cpp:96-131): 5 magic bytes "MILO1",
// u32 LE header length, a JSON header, a little-endian payload.
//  * packed-i3 (pack.cpp:306-400): words (or plane A then plane B) as u32,
//    binary16 scales, binary16 zeros (asymmetric only); validated like
//    load_packed (dtype, names, exact payload size).
//  * compensator factors written by quantize (pipeline.cpp:233-283; the
//    reference has no reader): symm-i3 = u8 codes + binary16 scales per
//    (row, 64-group), U (k x r) and V^T (n x r, "transposed"); real = f32 U
//    (k x r) and V (r x n).
// ===========================================================================
namespace {

// Flat JSON object (strings, integers, booleans); nested values are skipped.
struct JsonFlat {
  std::map<std::string, std::string> str;
  std::map<std::string, long long> num;
  std::map<std::string, bool> boolean;
};

bool json_flat_parse(const std::string& t, JsonFlat& out) {
  size_t i = 0;
  auto ws = [&] {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\t' || t[i] == '\r')) ++i;
  };
  auto str = [&](std::string& s) -> bool {
    if (i >= t.size() || t[i] != '"') return false;
    ++i;
    s.clear();
    while (i < t.size() && t[i] != '"') {
      if (t[i] == '\\' && i + 1 < t.size()) {
        ++i;
        s.push_back(t[i] == 'n' ? '\n' : t[i] == 't' ? '\t' : t[i]);
      } else {
        s.push_back(t[i]);
      }
      ++i;
    }
    if (i >= t.size()) return false;
    ++i;
    return true;
  };
  std::function<bool()> skip_value = [&]() -> bool {  // nested objects / arrays
    ws();
    if (i >= t.size()) return false;
    if (t[i] == '"') {
      std::string s;
      return str(s);
    }
    if (t[i] == '{' || t[i] == '[') {
      const char close = t[i] == '{' ? '}' : ']';
      ++i;
      ws();
      if (i < t.size() && t[i] == close) {
        ++i;
        return true;
      }
      for (;;) {
        if (close == '}') {
          ws();
          std::string k;
          if (!str(k)) return false;
          ws();
          if (i >= t.size() || t[i] != ':') return false;
          ++i;
        }
        if (!skip_value()) return false;
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == close) {
          ++i;
          return true;
        }
        return false;
      }
    }
    while (i < t.size() && t[i] != ',' && t[i] != '}' && t[i] != ']') ++i;
    return true;
  };
  ws();
  if (i >= t.size() || t[i] != '{') return false;
  ++i;
  ws();
  if (i < t.size() && t[i] == '}') return true;
  for (;;) {
    ws();
    std::string key;
    if (!str(key)) return false;
    ws();
    if (i >= t.size() || t[i] != ':') return false;
    ++i;
    ws();
    if (i >= t.size()) return false;
    if (t[i] == '"') {
      std::string v;
      if (!str(v)) return false;
      out.str[key] = v;
    } else if (t.compare(i, 4, "true") == 0) {
      out.boolean[key] = true;
      i += 4;
    } else if (t.compare(i, 5, "false") == 0) {
      out.boolean[key] = false;
      i += 5;
    } else if (t[i] == '-' || (t[i] >= '0' && t[i] <= '9')) {
      size_t j = i;
      while (j < t.size() && (t[j] == '-' || t[j] == '+' || t[j] == '.' || t[j] == 'e' || t[j] == 'E' ||
                              (t[j] >= '0' && t[j] <= '9')))
        ++j;
      out.num[key] = std::atoll(t.substr(i, j - i).c_str());
      i = j;
    } else if (!skip_value()) {
      return false;
    }
    ws();
    if (i < t.size() && t[i] == ',') {
      ++i;
      continue;
    }
    if (i < t.size() && t[i] == '}') return true;
    return false;
  }
}

milo_status read_container(const char* path, JsonFlat& h, std::vector<uint8_t>& payload) {
  FILE* f = path ? std::fopen(path, "rb") : nullptr;
  if (!f) return fail(MILO_ERR_IO, "cannot open '%s' for reading", path ? path : "(null)");
  std::vector<uint8_t> all;
  uint8_t buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) all.insert(all.end(), buf, buf + n);
  std::fclose(f);
  if (all.size() < 5 || std::memcmp(all.data(), "MILO1", 5) != 0)
    return fail(MILO_ERR_FORMAT, "'%s': bad magic, not a MILO1 container", path);
  if (all.size() < 9) return fail(MILO_ERR_FORMAT, "container truncated while reading header length");
  const uint32_t hlen = (uint32_t)all[5] | ((uint32_t)all[6] << 8) | ((uint32_t)all[7] << 16) | ((uint32_t)all[8] << 24);
  if (all.size() < 9 + (size_t)hlen) return fail(MILO_ERR_FORMAT, "'%s': truncated header", path);
  const std::string header(reinterpret_cast<const char*>(all.data() + 9), hlen);
  if (!json_flat_parse(header, h)) return fail(MILO_ERR_FORMAT, "'%s': bad container header", path);
  payload.assign(all.begin() + 9 + hlen, all.end());
  return MILO_OK;
}

bool json_get(const JsonFlat& h, const char* k, long long& v) {
  auto it = h.num.find(k);
  if (it == h.num.end()) return false;
  v = it->second;
  return true;
}

float host_half_to_float(uint16_t h) {
  const uint32_t s = (uint32_t)(h >> 15) << 31, e = (h >> 10) & 31, m = h & 1023;
  uint32_t bits;
  if (e == 0) {
    if (m == 0) {
      bits = s;
    } else {  // subnormal
      int ee = -1;
      uint32_t mm = m;
      do {
        ++ee;
        mm <<= 1;
      } while (!(mm & 1024));
      bits = s | ((uint32_t)(127 - 15 - ee) << 23) | ((mm & 1023) << 13);
    }
  } else if (e == 31) {
    bits = s | 0x7F800000u | (m << 13);
  } else {
    bits = s | ((e + 127 - 15) << 23) | (m << 13);
  }
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

// Owned host copy of a loaded packed-i3 container behind a milo_packed_desc.
struct PackedHost {
  milo_packed_desc d{};
  std::vector<uint32_t> words, pa, pb;
  std::vector<uint16_t> scales, zeros;
};

milo_status load_packed_host(const char* path, PackedHost& P) {
  JsonFlat h;
  std::vector<uint8_t> pl;
  milo_status st = read_container(path, h, pl);
  if (st != MILO_OK) return st;
  auto dt = h.str.find("dtype");
  if (dt == h.str.end() || dt->second != "packed-i3") return fail(MILO_ERR_FORMAT, "'%s': dtype is not packed-i3", path);
  long long rows, cols, gs;
  auto lay = h.str.find("layout");
  auto mode = h.str.find("mode");
  auto split = h.boolean.find("split");
  if (!json_get(h, "rows", rows) || !json_get(h, "cols", cols) || !json_get(h, "group_size", gs) ||
      lay == h.str.end() || mode == h.str.end() || split == h.boolean.end())
    return fail(MILO_ERR_FORMAT, "'%s': bad container header", path);
  int layout;
  if (lay->second == "linear") layout = MILO_LAYOUT_LINEAR;
  else if (lay->second == "tiled16x64") layout = MILO_LAYOUT_TILED16X64;
  else return fail(MILO_ERR_FORMAT, "unknown pack layout '%s'", lay->second.c_str());
  int md;
  if (mode->second == "symmetric") md = MILO_MODE_SYMMETRIC;
  else if (mode->second == "asymmetric") md = MILO_MODE_ASYMMETRIC;
  else return fail(MILO_ERR_FORMAT, "unknown dequant mode '%s'", mode->second.c_str());
  if (rows <= 0 || cols <= 0 || gs <= 0 || (rows * cols) % 32 != 0 || (rows * cols) % gs != 0)
    return fail(MILO_ERR_FORMAT, "'%s': inconsistent shape in header", path);
  const size_t groups = (size_t)(rows * cols / 32), nw = groups * 3, qg = (size_t)(rows * cols / gs);
  const size_t expect = nw * 4 + qg * 2 + (md == MILO_MODE_ASYMMETRIC ? qg * 2 : 0);
  if (pl.size() != expect)
    return fail(MILO_ERR_FORMAT, "'%s': payload is %zu bytes, expected %zu", path, pl.size(), expect);
  const uint8_t* p = pl.data();
  const bool sp = split->second;
  if (sp) {
    P.pa.resize(groups * 2);
    P.pb.resize(groups);
    std::memcpy(P.pa.data(), p, groups * 8);
    std::memcpy(P.pb.data(), p + groups * 8, groups * 4);
  } else {
    P.words.resize(nw);
    std::memcpy(P.words.data(), p, nw * 4);
  }
  p += nw * 4;
  P.scales.resize(qg);
  std::memcpy(P.scales.data(), p, qg * 2);
  p += qg * 2;
  if (md == MILO_MODE_ASYMMETRIC) {
    P.zeros.resize(qg);
    std::memcpy(P.zeros.data(), p, qg * 2);
  }
  milo_packed_desc& d = P.d;
  d.rows = (uint64_t)rows;
  d.cols = (uint64_t)cols;
  d.layout = layout;
  d.split = sp ? 1 : 0;
  d.mode = md;
  d.group_size = (uint64_t)gs;
  d.words = P.words.empty() ? nullptr : P.words.data();
  d.n_words = P.words.size();
  d.plane_a = P.pa.empty() ? nullptr : P.pa.data();
  d.n_plane_a = P.pa.size();
  d.plane_b = P.pb.empty() ? nullptr : P.pb.data();
  d.n_plane_b = P.pb.size();
  d.scales = P.scales.data();
  d.n_scales = P.scales.size();
  d.zeros = P.zeros.empty() ? nullptr : P.zeros.data();
  d.n_zeros = P.zeros.size();
  return MILO_OK;
}

struct FactorHost {
  long long rows = 0, cols = 0, rank = 0, gs = 64;
  bool transposed = false, real = false;
  std::vector<uint8_t> codes;
  std::vector<float> scales, values;
};

milo_status load_factor(const char* path, FactorHost& F) {
  JsonFlat h;
  std::vector<uint8_t> pl;
  milo_status st = read_container(path, h, pl);
  if (st != MILO_OK) return st;
  auto dt = h.str.find("dtype");
  if (dt == h.str.end() || !json_get(h, "rows", F.rows) || !json_get(h, "cols", F.cols) ||
      !json_get(h, "rank", F.rank) || F.rows <= 0 || F.cols <= 0 || F.rank < 0)
    return fail(MILO_ERR_FORMAT, "'%s': bad compensator header", path);
  if (dt->second == "symm-i3") {
    if (!json_get(h, "group_size", F.gs) || F.gs <= 0) return fail(MILO_ERR_FORMAT, "'%s': bad group_size", path);
    auto tr = h.boolean.find("transposed");
    F.transposed = tr != h.boolean.end() && tr->second;
    const size_t n = (size_t)(F.rows * F.cols), gpr = (size_t)((F.cols + F.gs - 1) / F.gs);
    if (pl.size() != n + (size_t)F.rows * gpr * 2)
      return fail(MILO_ERR_FORMAT, "'%s': payload is %zu bytes, expected %zu", path, pl.size(), n + (size_t)F.rows * gpr * 2);
    F.codes.assign(pl.begin(), pl.begin() + n);
    F.scales.resize((size_t)F.rows * gpr);
    for (size_t i = 0; i < F.scales.size(); ++i)
      F.scales[i] = host_half_to_float((uint16_t)(pl[n + 2 * i] | (pl[n + 2 * i + 1] << 8)));
  } else if (dt->second == "f32") {
    F.real = true;
    const size_t n = (size_t)(F.rows * F.cols);
    if (pl.size() != n * 4) return fail(MILO_ERR_FORMAT, "'%s': payload is %zu bytes, expected %zu", path, pl.size(), n * 4);
    F.values.resize(n);
    std::memcpy(F.values.data(), pl.data(), n * 4);
  } else {
    return fail(MILO_ERR_FORMAT, "'%s': dtype '%s' is not a compensator factor", path, dt->second.c_str());
  }
  return MILO_OK;
}

}  // namespace

extern "C" {

milo_status milo_packed_load_host(const char* path, milo_packed_desc* desc, void** handle) {
  if (!desc || !handle) return fail(MILO_ERR_ARGUMENT, "null argument");
  *handle = nullptr;
  PackedHost* P = new PackedHost();
  milo_status st = load_packed_host(path, *P);
  if (st != MILO_OK) {
    delete P;
    return st;
  }
  *desc = P->d;
  *handle = P;
  return MILO_OK;
}

void milo_packed_host_free(void* handle) { delete static_cast<PackedHost*>(handle); }

milo_status milo_weight_load(const char* path, milo_weight** out) {
  if (!out) return fail(MILO_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  PackedHost P;
  milo_status st = load_packed_host(path, P);
  if (st != MILO_OK) return st;
  return milo_weight_create(&P.d, out);
}

milo_status milo_comp_load(const char* u_path, const char* v_path, milo_comp** out) {
  if (!out) return fail(MILO_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  FactorHost U, V;
  milo_status st = load_factor(u_path, U);
  if (st == MILO_OK) st = load_factor(v_path, V);
  if (st != MILO_OK) return st;
  if (U.real != V.real || U.rank != V.rank) return fail(MILO_ERR_FORMAT, "compensator factors disagree (storage / rank)");
  milo_comp_desc d{};
  d.rank = (uint64_t)U.rank;
  if (U.real) {  // U: k x r, V: r x n
    if (U.cols != U.rank || V.rows != V.rank) return fail(MILO_ERR_SHAPE, "compensator factor shapes do not match the rank");
    d.rows = (uint64_t)U.rows;
    d.cols = (uint64_t)V.cols;
    d.storage = MILO_COMP_REAL;
    d.U = U.values.data();
    d.V = V.values.data();
  } else {  // qU: k x r, qVt: n x r (transposed)
    if (U.cols != U.rank || V.cols != V.rank || !V.transposed || U.gs != V.gs)
      return fail(MILO_ERR_SHAPE, "symm-i3 compensator factor shapes do not match the rank");
    d.rows = (uint64_t)U.rows;
    d.cols = (uint64_t)V.rows;
    d.storage = MILO_COMP_SYMM_INT3;
    d.qu_codes = U.codes.data();
    d.qu_scales = U.scales.data();
    d.qvt_codes = V.codes.data();
    d.qvt_scales = V.scales.data();
    d.group_size = (uint64_t)U.gs;
  }
  return milo_comp_create(&d, out);
}

}  // extern "C"

// Expert-parallel layer over NCCL (include/milo_b200.h milo_ep_*).
#include "ep_nccl.cuh"
