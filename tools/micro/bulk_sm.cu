// Per-SM throughput of 1D cp.async.bulk copies from L2-resident data into shared
// memory: one CTA per SM, one thread keeps `slots` copies of `chunk` bytes in flight.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory"); }
__device__ int g_spin;
__device__ __forceinline__ void waitp(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  if (g_spin) {
    do { asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory"); } while (!ok);
  } else {
    do { asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory"); } while (!ok);
  }
}
__device__ int g_lanes;
__global__ void k(const uint8_t* src, size_t src_bytes, int chunk, int slots, int iters, int pieces, long long* cyc) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int L = g_lanes;
  const int lane = threadIdx.x & 31;
  if (lane >= L) return;
  const int warp = (threadIdx.x >> 5) * L + lane;  // issuer id
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  uint8_t* ring = smem + 1024 + (size_t)warp * slots * chunk;
  for (int s = 0; s < slots; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nchunks = src_bytes / chunk;
  long long t0 = clock64();
  uint32_t ph = 0;
  for (int i = 0; i < iters + slots; ++i) {
    const int s = i % slots;
    if (i >= slots) { waitp(&bars[s], ph); if (s == slots - 1) ph ^= 1; }
    if (i < iters) {
      expect(&bars[s], chunk);
      const uint8_t* p = src + ((blockIdx.x * 7 + warp * 3 + i) % nchunks) * chunk;
      const int piece = chunk / pieces;
      for (int q = 0; q < pieces; ++q) bulk(ring + s * chunk + q * piece, p + q * piece, piece, &bars[s]);
    }
  }
  if (warp == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  uint8_t* src; long long* cyc; cudaMalloc(&src, 4 << 20); cudaMemset(src, 1, 4 << 20); cudaMalloc(&cyc, 8 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int L : {1, 4}) {
  int spin = 1;
  cudaMemcpyToSymbol(g_spin, &spin, 4);
  cudaMemcpyToSymbol(g_lanes, &L, 4);
  printf("-- issuers per warp: %d\n", L);
  for (int nw : {1, 2})
    for (int chunk : {4096, 16384})
      for (int slots : {2, 4}) {
        const int pieces = 1;
        if ((size_t)chunk * slots * nw * L > 190 * 1024) continue;
        const int iters = 1000;
        k<<<sms, 32 * nw, 1024 + chunk * slots * nw * L>>>(src, 4 << 20, chunk, slots, iters, pieces, cyc);
        cudaDeviceSynchronize();
        long long h[256]; cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
        double mx = 0; for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("warps %d chunk %6d slots %d: %.1f B/clk/SM (%.0f GB/s/SM)  %.0f cycles per copy per warp %s\n", nw, chunk, slots,
               (double)chunk * iters * nw * L / mx, (double)chunk * iters * nw * L / mx * 1.965, mx / iters,
               cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
