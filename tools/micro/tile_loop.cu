// Cycles per macro tile of the decode kernel's inner loop (tile_real) on
// smem-resident tiles, W warps on one SM: isolates the dequant + MMA issue rate
// from the rest of the kernel.  nvcc -arch=sm_100a -O3 -I../../paper_2504_02658_b200/csrc
#include <cstdio>
#include "decode.cuh"
using namespace milo_dev;
template <int NT, int NMAT, int NA>
__device__ __forceinline__ void tile_nomma(const uint8_t* tile0, int mstride, const BTile<NT>& b,
                                           float (&acc)[NA][4][NT][4], const DqConsts& dq, int lane) {
  const int q = lane & 3;
#pragma unroll
  for (int mat = 0; mat < NMAT; ++mat) {
    const uint8_t* tile = tile0 + mat * mstride;
    const uint4 pa = *reinterpret_cast<const uint4*>(tile + kPlaneAOff + lane * 16);
    const uint2 pb = *reinterpret_cast<const uint2*>(tile + kPlaneBOff + lane * 8);
    const uint4 m0 = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32);
    const uint4 m1 = *reinterpret_cast<const uint4*>(tile + kMetaOff + q * 32 + 16);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint4 mm = j == 0 ? m0 : m1;
      const uint32_t S[2] = {mm.x, mm.z}, O[2] = {mm.y, mm.w};
      uint32_t wv[16];
      unit_dequant(j == 0 ? pa.x : pa.z, j == 0 ? pa.y : pa.w, j == 0 ? pb.x : pb.y, S, O, dq, wv);
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[mat][i & 3][0][(i >> 2)] += __uint_as_float(wv[i] ^ b.v[j][0][0]);
    }
  }
}
template <int NMAT, bool MMA>
__global__ void __launch_bounds__(512, 1) k_tiles(float* out, int iters, long long* cyc, int mode) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4 * 2 * kTileBytes; i += blockDim.x) sm[i] = (uint8_t)(i * 37 + 11);
  if (threadIdx.x < 2 * 32 * 4) {  // sane binary16 (s, off) pairs in the meta section
    const int t = threadIdx.x / 32, m = (threadIdx.x / 32) % 2;
    (void)t; (void)m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 2; i += blockDim.x) {
    __half2* meta = reinterpret_cast<__half2*>(sm + i * kTileBytes + kMetaOff);
    for (int j = 0; j < 64; ++j) meta[j] = __floats2half2_rn(0.01f, -0.02f);
  }
  __syncthreads();
  const DqConsts dq = make_dq_consts(mode);
  BTile<1> b;
  b.v[0][0][0] = b.v[0][0][1] = b.v[1][0][0] = b.v[1][0][1] = 0x3c003c00u ^ lane;
  float acc[NMAT][4][1][4] = {};
  const uint8_t* base = sm + (warp & 1) * 4 * kTileBytes * NMAT / 2;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int kk = 0; kk < 4; ++kk)
      if (MMA) tile_real<1, NMAT, NMAT>(base + kk * kTileBytes, 4 * kTileBytes, b, acc, dq, lane);
      else tile_nomma<1, NMAT, NMAT>(base + kk * kTileBytes, 4 * kTileBytes, b, acc, dq, lane);
  }
  long long t1 = clock64();
  float s = 0;
  for (int x = 0; x < NMAT; ++x)
    for (int i = 0; i < 4; ++i)
      for (int e = 0; e < 4; ++e) s += acc[x][i][0][e];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64);
  const int iters = 512;
  cudaFuncSetAttribute(k_tiles<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  cudaFuncSetAttribute(k_tiles<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  cudaFuncSetAttribute(k_tiles<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  cudaFuncSetAttribute(k_tiles<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  for (int mma = 0; mma <= 1; ++mma)
  for (int nm = 1; nm <= 2; ++nm)
    for (int w : {8, 16}) {
      auto k = mma ? (nm == 2 ? k_tiles<2, true> : k_tiles<1, true>) : (nm == 2 ? k_tiles<2, false> : k_tiles<1, false>);
      k<<<1, 32 * w, 64 << 10>>>(out, iters, cyc, 1);
      k<<<1, 32 * w, 64 << 10>>>(out, iters, cyc, 1);
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double tiles_per_smsp = (double)iters * 4 * nm * w / 4;
      printf("mma=%d NMAT=%d warps=%2d (%d/SMSP): %.1f cycles per tile per SMSP  %s\n", mma, nm, w, w / 4, c / tiles_per_smsp,
             cudaGetErrorString(e));
    }
  return 0;
}
