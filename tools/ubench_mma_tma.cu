// Microbenchmark: tcgen05.mma (M128 N32 K16, SS, 8 per 128x32x128 tile) throughput
// while one warp streams 32 KB bulk copies global(L2-resident) -> SMEM at full
// rate: SMEM-port interference between the TMA writes and the MMA operand reads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma_tma tools/ubench_mma_tma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
constexpr int kStages = 4;
__global__ void __launch_bounds__(128, 1) k(int iters, int tma_on, int mma_on, const uint8_t* src, size_t src_bytes,
                                            unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  // [0, 40K): MMA operands (A 32K + B 8K); [40K, 40K + 4*32K): TMA stages
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, full[kStages];
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40960 / 4; i += blockDim.x) ((uint32_t*)buf)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const int N = 32;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t a0 = smem_u32(buf), b0 = smem_u32(buf + 32768);
  if (warp == 0) {
    long long t0 = clock64();
    if (mma_on) {
      for (int it = 0; it < iters; ++it)
        for (int kb = 0; kb < 2; ++kb)
          for (int ks = 0; ks < 4; ++ks)
            mma_warp(tm + (uint32_t)((it % 8) * N), sdesc(a0 + kb * 16384 + ks * 32), sdesc(b0 + kb * N * 128 + ks * 32),
                     idesc, (kb | ks) != 0);
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar)));
      while (!try_wait(smem_u32(&bar), 0)) {}
    } else {
      while (clock64() - t0 < 3000000) {}
    }
    long long t1 = clock64();
    if (lane == 0) {
      done = 1;
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
  } else if (warp == 1 && tma_on) {
    // stream 32 KB chunks into kStages stages, waiting for each stage's previous fill
    unsigned long long n = 0;
    const size_t chunks = src_bytes / 32768;
    long long t0 = clock64();
    uint32_t ph[kStages] = {0};
    for (int s = 0; s < kStages; ++s) {
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32768));
        const uint8_t* g = src + ((blockIdx.x * 7 + n) % chunks) * 32768;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(buf + 40960 + s * 32768)), "l"(g), "r"(32768), "r"(smem_u32(&full[s])) : "memory");
      }
      ++n;
    }
    for (int s = 0; !done; s = (s + 1) % kStages) {
      while (!try_wait(smem_u32(&full[s]), ph[s])) {}
      ph[s] ^= 1;
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32768));
        const uint8_t* g = src + ((blockIdx.x * 7 + n) % chunks) * 32768;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(buf + 40960 + s * 32768)), "l"(g), "r"(32768), "r"(smem_u32(&full[s])) : "memory");
      }
      ++n;
    }
    for (int s = 0; s < kStages; ++s) { while (!try_wait(smem_u32(&full[s]), ph[s])) {} }
    long long t1 = clock64();
    if (blockIdx.x == 0 && lane == 0) { out[1] = n; out[2] = t1 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 8);
  const size_t src_bytes = 16u << 20;     // 16 MB: L2-resident
  uint8_t* src; cudaMalloc(&src, src_bytes); cudaMemset(src, 0, src_bytes);
  const int smem = 40960 + kStages * 32768 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct C { int tma, mma; } cs[] = {{0, 1}, {1, 0}, {1, 1}};
  for (auto c : cs) {
    const int iters = 4000;
    cudaMemset(d, 0, 64);
    k<<<148, 128, smem>>>(iters, c.tma, c.mma, src, src_bytes, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("tma %d mma %d: MMA %7.1f cycles/tile; TMA %.1f B/cycle per SM (%.2f TB/s chip @1.965GHz)\n", c.tma, c.mma,
           c.mma ? (double)h[0] / iters : 0.0, h[2] ? (double)h[1] * 32768 / h[2] : 0.0,
           h[2] ? (double)h[1] * 32768 / h[2] * 148 * 1.965e9 / 1e12 : 0.0);
  }
  return 0;
}
