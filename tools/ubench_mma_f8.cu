// Microbenchmark: cycles per 128-token tile (d = 128) of the fused kernel's MMA,
// bf16 kind::f16 (8 x K16) vs e4m3 kind::f8f6f4 (4 x K32), N = 32 columns,
// straight-line warp-uniform issue + two commits per tile, D slot rotating over 16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma_f8 tools/ubench_mma_f8.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <bool F8>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (F8)
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
template <bool F8, int KS>
__global__ void __launch_bounds__(128, 1) k(int iters, int N, int wait_each, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)buf)[i] = F8 ? 0x38383838u : 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
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
  const uint32_t fmt = F8 ? 0u : ((1u << 7) | (1u << 10));
  const uint32_t idesc = (1u << 4) | fmt | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t a0 = smem_u32(buf), b0 = smem_u32(buf + 32768);
  const uint64_t hi = ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
  const uint32_t alo = ((a0 >> 4) & 0x3FFF) | (1u << 16), blo = ((b0 >> 4) & 0x3FFF) | (1u << 16);
  unsigned long long t0 = clock64();
  uint32_t ph = 0;
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tm + (uint32_t)((it % 16) * N);
#pragma unroll
      for (int j = 0; j < KS; ++j) {
        const uint32_t kb = j / 4, ks = j % 4;
        mma<F8>(d, hi | (alo + kb * 1024 + ks * 2), hi | (blo + kb * N * 8 + ks * 2), idesc, j > 0);
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar[0])));
      if (wait_each) {
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(&bar[0])), "r"(ph));
        ph ^= 1;
      }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar[1])));
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar[1])));
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <bool F8, int KS>
void run(const char* name, int N, int wait_each) {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k<F8, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  const int iters = 4000;
  k<F8, KS><<<148, 128, 100000>>>(iters, N, wait_each, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-6s N %3d wait_each %d: %7.1f cycles per tile, %6.1f per MMA\n", name, N, wait_each, (double)h / iters,
         (double)h / iters / KS);
  cudaFree(d);
}
int main() {
  for (int w = 0; w < 2; ++w) {
    run<false, 8>("bf16", 32, w);
    run<true, 4>("e4m3", 32, w);
    run<true, 4>("e4m3", 64, w);
    run<false, 8>("bf16", 64, w);
  }
  return 0;
}
