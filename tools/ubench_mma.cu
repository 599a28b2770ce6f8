// Microbenchmark: tcgen05.mma kind::f16 throughput for M=128, N in {16,32,64,128,256}, K=16, SS operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma tools/ubench_mma.cu
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
__global__ void __launch_bounds__(128, 1) k(int iters, int N, unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t cbar[2];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)buf)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[1])));
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
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(buf), b0 = smem_u32(buf + 32768);
    for (int it = 0; it < iters; ++it) {
      for (int kb = 0; kb < 2; ++kb)
        for (int ks = 0; ks < 4; ++ks) {
          uint64_t a = sdesc(a0 + kb * 16384 + ks * 32), b = sdesc(b0 + kb * N * 128 + ks * 32);
          uint32_t acc = (kb | ks) != 0;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                       ::"r"(tm + (uint32_t)((it % (512 / N)) * N)), "l"(a), "l"(b), "r"(idesc), "r"(acc));
        }
      if (mode >= 1) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&cbar[0])));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&cbar[1])));
      }
      if (mode >= 2) asm volatile("tcgen05.fence::after_thread_sync;");
      if (mode >= 3) {   // wait for this tile's MMAs to finish (serialised tiles)
        const uint32_t par = it & 1;
        asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(smem_u32(&cbar[0])), "r"(par));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
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
  for (int mode = 0; mode < 4; ++mode)
  for (int N : {32, 64}) {
    const int iters = 2000;
    k<<<148, 128, 100000>>>(iters, N, d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("N %d err %s\n", N, cudaGetErrorString(e)); return 1; }
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d N %3d: %.1f cycles per MMA (M=128,K=16), %.1f cycles per 128x%dx128 tile\n", mode, N, (double)h / (iters * 8), (double)h / iters, N);
  }
  return 0;
}
