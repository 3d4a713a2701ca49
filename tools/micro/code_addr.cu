// Is a __device__ function's address a readable global address (so its code can be L2-prefetched)?
#include <cstdio>
#include <cstdint>
__device__ __noinline__ float far_fn(float a) { return a / (1.0f + expf(-a)) * 3.0f + sinf(a); }
__global__ void k(unsigned long long* out, float x) {
  float (*fp)(float) = far_fn;
  const unsigned long long addr = (unsigned long long)fp;
  out[0] = addr;
  unsigned long long v = 0;
  asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(addr));
  out[1] = v;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(addr & ~255ull));
  out[2] = __float_as_uint(fp(x));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  k<<<1, 1>>>(d, 1.5f);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[3] = {};
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("err=%s addr=%llx first8=%016llx\n", cudaGetErrorString(e), h[0], h[1]);
  return 0;
}
