// Per-SM cp.async.bulk throughput, global -> shared: `issuers` threads per CTA (one per warp),
// each keeping `slots` copies of `chunk` bytes in flight; source L2-resident (4 MB) or
// HBM-streamed (1 GB).  One CTA per SM.  Prints B/clk/SM and the implied per-SM GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint8_t* src, size_t src_bytes, int chunk, int slots, int iters, long long* cyc, int pieces) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + w * 16;
  uint8_t* ring = smem + 2048 + (size_t)w * slots * chunk;
  if (lane == 0) {
    for (int s = 0; s < slots; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const size_t nchunks = src_bytes / chunk;
  long long t0 = clock64();
  uint32_t ph = 0;
  if (lane == 0) {
    for (int i = 0; i < iters + slots; ++i) {
      const int s = i % slots;
      if (i >= slots) {
        uint32_t ok;
        do {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(su32(&bars[s])), "r"(ph) : "memory");
        } while (!ok);
        if (s == slots - 1) ph ^= 1;
      }
      if (i < iters) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(chunk) : "memory");
        const size_t idx = ((size_t)blockIdx.x * nw * iters + (size_t)w * iters + i) % nchunks;
        const int pc = chunk / pieces;
        for (int q = 0; q < pieces; ++q)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su32(ring + s * chunk + q * pc)), "l"(src + idx * chunk + q * pc), "r"(pc), "r"(su32(&bars[s])) : "memory");
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  uint8_t* src; long long* cyc;
  const size_t big = (size_t)1 << 30;
  cudaMalloc(&src, big); cudaMemset(src, 1, big); cudaMalloc(&cyc, 8 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (size_t sb : {(size_t)4 << 20, big})
    for (int nw : {1, 4})
      for (int chunk : {4096, 16384})
        for (int slots : {2, 8})
          for (int pieces : {1, 2, 4, 8}) {
          if ((size_t)chunk * slots * nw > 200 * 1024) continue;
          const int iters = sb == big ? 200 : 400;
          k<<<sms, 32 * nw, 2048 + chunk * slots * nw>>>(src, sb, chunk, slots, iters, cyc, pieces);
          cudaDeviceSynchronize();
          long long h[256]; cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
          double mx = 0; for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
          const double bpc = (double)chunk * iters * nw / mx;
          printf("%s issuers %2d chunk %6d slots %d pieces %d: %6.1f B/clk/SM  %6.0f clk/slot/issuer %s\n",
                 sb == big ? "HBM" : "L2 ", nw, chunk, slots, pieces, bpc, mx / iters, cudaGetErrorString(cudaGetLastError()));
        }
  return 0;
}
