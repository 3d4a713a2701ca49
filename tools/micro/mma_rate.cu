// tcgen05.mma issue / completion rate, one CTA per SM, one issuing thread:
// M = 128, K = 16 (kind::f16), N in {16..256}, A from TMEM (ts) or shared memory (ss).
// Prints cycles per MMA for issue (back-to-back, no waits) and to completion
// (commit + mbarrier wait after the batch).  Operand contents are garbage (zeros).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/mma_rate tools/micro/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)64u << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ uint32_t idesc(int n) { return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }

template <bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int n, int iters, long long* out, int issuers, int per = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t ring[8];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(issuers));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if ((threadIdx.x & 31) == 0 && warp < issuers) {
    const uint32_t id = idesc(n);
    const uint64_t da = desc_sw128(smem_u32(base));
    const uint64_t db = desc_sw128(smem_u32(base + 32768));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)(warp * 64);  // one accumulator per issuing warp
      if (TS)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                     "r"(tmem + 256u + (uint32_t)((i & 3) * 8)), "l"(db + 2 * (i & 3)), "r"(id), "r"(1));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(da + 2 * (i & 3)), "l"(db + 2 * (i & 3)), "r"(id), "r"(1));
      if (per > 0 && (i % per) == per - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&ring[(i / per) & 7]))
                     : "memory");
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t ok = warp != 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar))
                   : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0 && warp == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Stage-like loop: PER MMAs (ts, N = n) then a commit to a ring barrier, optionally
// waiting (already complete or not) on a barrier before each stage.
template <int PER, int WAIT>
__global__ void __launch_bounds__(128, 1) stage_rate(int n, int stages, long long* out) {
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t ring[8];
  __shared__ __align__(1024) uint8_t bsm[16384];
  __shared__ __align__(8) uint64_t plain;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&plain)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(&plain)) : "memory");
    const uint32_t id = idesc(n);
    const uint64_t db = desc_sw128(smem_u32(bsm));
    long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
      if ((WAIT & 1) && s >= 8) {  // the commit of stage s - 8 (long done, or the one 8 back)
        uint32_t ok = 0;
        const uint32_t par = ((s - 8) >> 3) & 1;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok)
                       : "r"(smem_u32(&ring[s & 7])), "r"(par)
                       : "memory");
      }
      if (WAIT & 2) asm volatile("tcgen05.fence::after_thread_sync;");
      if (WAIT & 4) {  // a plain mbarrier that completed long ago (software arrivals only)
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok)
                       : "r"(smem_u32(&plain))
                       : "memory");
      }
#pragma unroll
      for (int j = 0; j < PER; ++j)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(tmem + 256u + (uint32_t)((j & 3) * 8)), "l"(db + 2 * (j & 3)), "r"(id), "r"(1));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&ring[s & 7]))
                   : "memory");
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = 0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// The same stage loop (4 MMAs + commit) while NOISE other warps of the CTA run a
// dense HFMA2 / LOP3 loop (a stand-in for the prefill kernel's dequant warps).
template <int NOISE>
__global__ void __launch_bounds__(32 * (1 + NOISE), 1) noisy_rate(int n, int stages, long long* out, uint32_t seed) {
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t ring[8];
  __shared__ __align__(1024) uint8_t bsm[16384];
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      const uint32_t id = idesc(n);
      const uint64_t db = desc_sw128(smem_u32(bsm));
      long long t0 = clock64();
      for (int s = 0; s < stages; ++s) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                       "r"(tmem + 256u + (uint32_t)(j * 8)), "l"(db + 2 * j), "r"(id), "r"(1));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&ring[s & 7]))
                     : "memory");
      }
      long long t1 = clock64();
      done = 1;
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
  } else if (seed == 7) {  // tcgen05.st traffic: each noise warp rewrites 32 columns of its lane quarter
    const uint32_t q = (uint32_t)(warp & 3) * 32;
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 16 + i;
    long long t0 = clock64(), iters = 0;
    while (!done) {
      ++iters;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t col = 384u + (uint32_t)(((warp >> 2) * 8 + i) & 3) * 32;
        asm volatile(
            "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                tmem + (q << 16) + col),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
            "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
            : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (blockIdx.x == 0 && threadIdx.x == 32) out[1] = (clock64() - t0) / (iters > 0 ? iters : 1);
  } else {
    __half2 a = __float2half2_rn((float)(seed & 7)), b = __float2half2_rn(0.5f), c = __float2half2_rn(0.25f);
    uint32_t w = seed ^ threadIdx.x;
    while (!done) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        w = (w * 1664525u) + 1013904223u;
        a = __hfma2(a, b, c);
        b = __hfma2(b, c, a);
      }
    }
    if (threadIdx.x == 32 && w == 17u) out[1] = (long long)__half2float(a.x);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
template <int NOISE>
void run_noisy(long long* d, uint32_t seed = 3) {
  long long h[2];
  const int stages = 2048;
  for (int rep = 0; rep < 2; ++rep) noisy_rate<NOISE><<<148, 32 * (1 + NOISE)>>>(64, stages, d, seed);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("4 MMAs (ts N=64) + commit with %2d busy %s warps: %7.1f cyc/stage; %s\n", NOISE, seed == 7 ? "TMEM-store" : "ALU",
         (double)h[0] / stages, seed == 7 ? "" : "");
  if (seed == 7) printf("   per store warp: 8 x 16x256b.x4 stores + wait::st = %lld cycles\n", h[1]);
}

// The prefill kernel's issuer form: the whole warp runs the loop, elect.sync inside
// the asm picks the issuing lane (operands in uniform registers); per stage: PER
// MMAs and one commit, optionally a poll of a shared-memory counter (always ready).
template <int PER, int POLL>
__global__ void __launch_bounds__(128, 1) warp_rate(int n, int stages, long long* out) {
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t ring[8];
  __shared__ __align__(1024) uint8_t bsm[16384];
  __shared__ uint32_t ready;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    ready = 1u << 30;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t id = idesc(n);
    const uint64_t db = desc_sw128(smem_u32(bsm));
    long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
      if (POLL) {
        uint32_t v;
        do {
          asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&ready)) : "memory");
        } while (v <= (uint32_t)s);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
#pragma unroll
      for (int j = 0; j < PER; ++j)
        asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(tmem + 256u + (uint32_t)((j & 3) * 8)), "l"(db + 2 * (j & 3)), "r"(id), "r"(1));
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                       smem_u32(&ring[s & 7]))
                   : "memory");
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
template <int PER, int POLL>
void run_warp(long long* d, int n) {
  long long h[2];
  const int stages = 2048;
  for (int rep = 0; rep < 2; ++rep) warp_rate<PER, POLL><<<148, 128>>>(n, stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("warp-converged elect issuer: %d MMAs (ts N=%d) + commit%s: %7.1f cyc/stage\n", PER, n,
         POLL ? " + counter poll + fence" : "", (double)h[0] / stages);
}

template <int PER, int WAIT>
void run_stage(long long* d, int n) {
  long long h[2];
  const int stages = 2048;
  for (int rep = 0; rep < 2; ++rep) stage_rate<PER, WAIT><<<148, 128>>>(n, stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("stage loop: %d MMAs (ts N=%d) + commit%s%s%s: %7.1f cyc/stage = %6.1f cyc/mma\n", PER, n,
         (WAIT & 1) ? " + wait(commit of stage-8)" : "", (WAIT & 2) ? " + fence::after" : "",
         (WAIT & 4) ? " + wait(plain, complete)" : "", (double)h[0] / stages, (double)h[0] / stages / PER);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[2];
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(mma_rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  run_stage<4, 0>(d, 64);
  run_warp<4, 0>(d, 64);
  run_warp<4, 1>(d, 64);
  run_stage<8, 0>(d, 64);
  run_warp<8, 0>(d, 64);
  return 0;
  run_noisy<0>(d);
  run_noisy<1>(d, 7);
  run_noisy<4>(d, 7);
  run_noisy<8>(d, 7);
  run_noisy<12>(d, 7);
  run_stage<4, 0>(d, 64);
  run_stage<4, 1>(d, 64);
  run_stage<4, 2>(d, 64);
  run_stage<4, 3>(d, 64);
  run_stage<4, 4>(d, 64);
  run_stage<4, 5>(d, 64);
  run_stage<4, 6>(d, 64);
  run_stage<8, 3>(d, 64);
  run_stage<8, 7>(d, 64);
  return 0;
  for (int per : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) mma_rate<true><<<148, 128, smem>>>(64, iters, d, 1, per);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("commit every %d MMAs, ts N=64: issue %6.1f cyc/mma, complete %6.1f\n", per, (double)h[0] / iters,
           (double)h[1] / iters);
  }
  for (int issuers = 1; issuers <= 4; issuers *= 2)
  for (int ts = 1; ts >= 0; --ts)
    for (int n : {16, 32, 64, 128, 256}) {
      if (issuers > 1 && n > 64) continue;
      for (int rep = 0; rep < 2; ++rep) {
        if (ts)
          mma_rate<true><<<148, 128, smem>>>(n, iters, d, issuers);
        else
          mma_rate<false><<<148, 128, smem>>>(n, iters, d, issuers);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
      }
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("issuers %d %s N=%3d: issue %6.1f cyc/mma-of-one-thread, complete %6.1f (floor 128*N/256 = %d)\n", issuers, ts ? "ts" : "ss", n,
             (double)h[0] / iters, (double)h[1] / iters, 128 * n / 256);
      (void)0;
    }
  return 0;
}
