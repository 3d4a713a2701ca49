// Streams S MB with per-warp bulk-copy rings (12 warps x 3 slots x 3584 B) and reports
// event time and in-kernel span (globaltimer first start -> last end) under
// different L2 states: after a write flush, after a read flush, and warm.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory"); }
__device__ __forceinline__ bool tryw(uint64_t* b, uint32_t ph) { uint32_t ok; asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory"); return ok; }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void ring_kernel(const uint8_t* src, size_t bytes_per_warp, int chunk, int slots, unsigned long long* span) {
  extern __shared__ __align__(128) uint8_t smem[];
  if (threadIdx.x == 0) atomicMin(&span[0], gt());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  uint8_t* ring = smem + 4096 + (size_t)warp * slots * chunk;
  const uint8_t* base = src + ((size_t)blockIdx.x * nw + warp) * bytes_per_warp;
  const int n = (int)(bytes_per_warp / chunk);
  if (lane == 0) for (int s = 0; s < slots; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  int issued = 0;
  auto issue = [&](int s) { expect(&bars[s], chunk); bulk(ring + s * chunk, base + (size_t)issued * chunk, chunk, &bars[s]); ++issued; };
  if (lane == 0) for (int s = 0; s < slots && issued < n; ++s) issue(s);
  __syncwarp();
  float acc = 0.f; int slot = 0; uint32_t ph = 0;
  for (int u = 0; u < n; ++u) {
    { long long t0 = clock64(); while (!tryw(&bars[slot], ph)) { if (clock64() - t0 > 2000000000LL) __trap(); } }
    acc += reinterpret_cast<const float*>(ring + slot * chunk)[lane];
    __syncwarp();
    if (lane == 0 && issued < n) issue(slot);
    if (++slot == slots) { slot = 0; ph ^= 1; }
  }
  if (acc == 1234.5f) span[2] = 1;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&span[1], gt());
}
__global__ void read_kernel(const uint4* src, size_t n4, unsigned long long* sink) {
  uint32_t acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) { uint4 v = src[i]; acc ^= v.x ^ v.w; }
  if (acc == 0x12345) sink[2] = 1;
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  uint8_t* buf; unsigned long long* span; cudaMalloc(&buf, (size_t)3 << 30); cudaMalloc(&span, 64); cudaMemset(buf, 1, (size_t)3 << 30);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int nw = 12, slots = 3, chunk = 3584; const size_t smem = 4096 + (size_t)nw * slots * chunk;
  uint8_t* fl = buf + ((size_t)2 << 30);
  for (int mb : {26, 100, 155, 400, 1000}) {
    for (int fmode = 0; fmode < 3; ++fmode) {
      const size_t per_warp = ((size_t)mb << 20) / ((size_t)sms * nw) / chunk * chunk;
      float best = 1e9, bspan = 1e9;
      for (int it = 0; it < 4; ++it) {
        if (fmode == 0) cudaMemset(fl, it, (size_t)512 << 20);
        if (fmode == 1) { cudaMemset(fl, it, (size_t)512 << 20); read_kernel<<<sms * 8, 256>>>((const uint4*)(buf + ((size_t)1 << 30)), ((size_t)512 << 20) / 16, span); }
        unsigned long long init[2] = {~0ull, 0ull}; cudaMemcpy(span, init, 16, cudaMemcpyHostToDevice);
        cudaEventRecord(a); ring_kernel<<<sms, nw * 32, smem>>>(buf, per_warp, chunk, slots, span); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); unsigned long long h[2]; cudaMemcpy(h, span, 16, cudaMemcpyDeviceToHost);
        if (it > 0) { best = ms < best ? ms : best; float sp = (h[1] - h[0]) * 1e-6f; bspan = sp < bspan ? sp : bspan; }
      }
      const double bytes = (double)per_warp * sms * nw;
      printf("%5d MB flush=%s: event %.1f us (%.0f GB/s)  in-kernel span %.1f us (%.0f GB/s)\n", mb, fmode == 0 ? "write" : fmode == 1 ? "w+read" : "none ",
             best * 1e3, bytes / best / 1e6, bspan * 1e3, bytes / bspan / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
