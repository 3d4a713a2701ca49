// Issue throughput of the legacy warp MMA (HMMA.16816.F32), HFMA2 and LOP3 on one SM
// with W warps: cycles per instruction per SMSP.  nvcc -arch=sm_100a -O3 pipe_tput.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__global__ void k_mma(float* out, int iters, long long* cyc) {
  float acc[8][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_hfma2(float* out, int iters, long long* cyc) {
  __half2 v[8];
  for (int j = 0; j < 8; ++j) v[j] = __floats2half2_rn(threadIdx.x * 0.001f + j, j);
  const __half2 s = __floats2half2_rn(0.999f, 0.999f), o = __floats2half2_rn(0.001f, 0.001f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __hfma2(v[j], s, o);
  }
  long long t1 = clock64();
  float sum = 0;
  for (int j = 0; j < 8; ++j) sum += __low2float(v[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_lop3(float* out, int iters, long long* cyc) {
  uint32_t v[8];
  for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * (j + 1);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("lop3.b32 %0, %0, 0x70007, 0x64006400, 0xEA;" : "+r"(v[j]));
  }
  long long t1 = clock64();
  uint32_t sum = 0;
  for (int j = 0; j < 8; ++j) sum += v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)sum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
  const int iters = 4096;
  const char* names[3] = {"HMMA.16816.F32", "HFMA2", "LOP3"};
  for (int kind = 0; kind < 3; ++kind)
    for (int w : {1, 2, 4, 8, 16}) {
      void (*k)(float*, int, long long*) = kind == 0 ? k_mma : kind == 1 ? k_hfma2 : k_lop3;
      k<<<1, 32 * w>>>(out, iters, cyc);
      k<<<1, 32 * w>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double per_smsp = (double)iters * 8 * w / (w < 4 ? w : 4);  // instructions per SMSP (warp w on SMSP w%4)
      printf("%-16s warps=%2d  cycles=%8lld  cycles/instr/SMSP=%.2f\n", names[kind], w, c, c / per_smsp);
    }
  return 0;
}
