// Issue cost of 1D cp.async.bulk: one CTA per SM issues `n` copies of `chunk` bytes into
// distinct smem buffers, all completing on ONE mbarrier, then waits for it (spin on
// test_wait or try_wait).  Issuers: 1 thread, or `lanes` lanes of one warp issuing
// round-robin.  Repeated `iters` times.  Source L2-resident (8 MB) or HBM (1 GB).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint8_t* src, size_t src_bytes, int chunk, int n, int lanes, int iters, int spin,
                  long long* cyc) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  uint8_t* buf = smem + 128;
  const int lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const size_t nchunks = src_bytes / chunk;
  const long long t0 = clock64();
  uint32_t ph = 0;
  for (int it = 0; it < iters; ++it) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(chunk * n)
                   : "memory");
    __syncwarp();
    for (int c = lane; c < n; c += lanes) {
      if (lane >= lanes) break;
      const size_t idx = ((size_t)blockIdx.x * 977 + (size_t)it * n + c) % nchunks;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(buf + (size_t)c * chunk)),
          "l"(src + idx * chunk), "r"(chunk), "r"(su32(bar))
          : "memory");
    }
    uint32_t ok = 0;
    do {
      if (spin)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(su32(bar)), "r"(ph) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(su32(bar)), "r"(ph) : "memory");
    } while (!ok);
    ph ^= 1;
    __syncwarp();
  }
  if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  uint8_t* src;
  long long* cyc;
  const size_t big = (size_t)1 << 30;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  cudaMalloc(&cyc, 8 * 1024);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (size_t sb : {(size_t)8 << 20, big})
    for (int spin : {0, 1})
      for (int chunk : {1792, 14336})
        for (int n : {1, 2, 4, 8, 16})
          for (int lanes : {1, 16}) {
            if ((size_t)chunk * n > 200 * 1024) continue;
            if (lanes > n && lanes != 1) continue;
            const int iters = 100;
            k<<<sms, 32, 128 + chunk * n>>>(src, sb, chunk, n, lanes, iters, spin, cyc);
            cudaDeviceSynchronize();
            long long h[256];
            cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
            double mx = 0, sum = 0;
            for (int i = 0; i < sms; ++i) {
              mx = h[i] > mx ? h[i] : mx;
              sum += h[i];
            }
            printf("%s %s chunk %6d n %2d lanes %2d: %7.0f clk/round (mean %7.0f)  %6.1f B/clk/SM  %s\n",
                   sb == big ? "HBM" : "L2 ", spin ? "spin" : "try ", chunk, n, lanes, mx / iters, sum / sms / iters,
                   (double)chunk * n * iters / mx, cudaGetErrorString(cudaGetLastError()));
          }
  return 0;
}
