// Microbenchmark: tcgen05.mma issue cost, lane-0-only loop vs whole-warp loop with an elected issue.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma3 tools/ubench_mma3.cu
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
__device__ __forceinline__ void mma_lane(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// whole warp executes; one elected lane issues
__device__ __forceinline__ void mma_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__global__ void __launch_bounds__(128, 1) k(int iters, int N, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)buf)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
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
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  unsigned long long t0 = clock64();
  const uint32_t a0 = smem_u32(buf), b0 = smem_u32(buf + 32768);
  const uint32_t desc_hi = (uint32_t)(sdesc(0) >> 32);
  if (mode == 0 && threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it)
      for (int kb = 0; kb < 2; ++kb)
        for (int ks = 0; ks < 4; ++ks)
          mma_lane(tm + (uint32_t)((it % (512 / N)) * N), sdesc(a0 + kb * 16384 + ks * 32),
                   sdesc(b0 + kb * N * 128 + ks * 32), idesc, (kb | ks) != 0);
  } else if (mode == 1 && warp == 0) {
    for (int it = 0; it < iters; ++it)
      for (int kb = 0; kb < 2; ++kb)
        for (int ks = 0; ks < 4; ++ks)
          mma_warp(tm + (uint32_t)((it % (512 / N)) * N), sdesc(a0 + kb * 16384 + ks * 32),
                   sdesc(b0 + kb * N * 128 + ks * 32), idesc, (kb | ks) != 0);
  } else if (mode >= 3 && warp == 0) {
    // per-tile overheads of the real MMA loop: 3 = + two commits, 4 = + fence::after_thread_sync,
    // 5 = + two test_waits of completed barriers, 6 = + commit only every 4th tile
    __shared__ __align__(8) uint64_t cb[2];
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cb[0])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cb[1])));
    }
    __syncwarp();
    const uint32_t alo = ((a0 >> 4) & 0x3FFF) | (1u << 16), blo = ((b0 >> 4) & 0x3FFF) | (1u << 16);
    for (int it = 0; it < iters; ++it) {
      if (mode >= 5) {
        uint32_t ok;
        asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(1u) : "memory");
        if (!ok) asm volatile("trap;");
        asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(1u) : "memory");
        if (!ok) asm volatile("trap;");
      }
      if (mode >= 4) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tm + (uint32_t)((it % (512 / N)) * N);
#pragma unroll 1
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll 4
        for (int ks = 0; ks < 4; ++ks)
          mma_warp(d, ((uint64_t)desc_hi << 32) | (alo + kb * 1024 + ks * 2),
                   ((uint64_t)desc_hi << 32) | (blo + kb * N * 8 + ks * 2), idesc, (kb | ks) != 0);
      if (mode != 6 || (it & 3) == 3) {
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&cb[0])));
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&cb[1])));
      }
    }
  } else if (mode == 2 && warp == 0) {
    // precomputed low words, 64-bit descriptors built by adding to the low word
    const uint32_t alo = ((a0 >> 4) & 0x3FFF) | (1u << 16), blo = ((b0 >> 4) & 0x3FFF) | (1u << 16);
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tm + (uint32_t)((it % (512 / N)) * N);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_warp(d, ((uint64_t)desc_hi << 32) | (alo + kb * 1024 + ks * 2),
                   ((uint64_t)desc_hi << 32) | (blo + kb * N * 8 + ks * 2), idesc, (kb | ks) != 0);
    }
  }
  if (warp == 0) {
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int mode = 0; mode < 7; ++mode)
    for (int N : {32}) {
      const int iters = 4000;
      k<<<148, 128, 100000>>>(iters, N, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("mode %d N %3d: %6.1f cycles per M128 K16 MMA\n", mode, N, (double)h / (iters * 8));
    }
  return 0;
}
