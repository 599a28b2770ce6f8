// Microbenchmark: tcgen05.mma kind::f16 shapes for the token-importance contraction.
//   SS  M128 N{32,64,256}: A (K tile) and B (Q) from SMEM
//   TS  M128 N32: A from TMEM, B from SMEM
//   SS  M64  N256: Q as A (padded to 64 rows), K tile as B (256 tokens)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma2 tools/ubench_mma2.cu
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
// kind: 0 SS, 1 TS (A in TMEM)
__global__ void __launch_bounds__(128, 1) k(int iters, int M, int N, int kind, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 131072 / 4; i += 128) ((uint32_t*)buf)[i] = 0x3c003c00u;
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
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(buf), b0 = smem_u32(buf + 65536);
    const int dslots = kind == 1 ? (384 / N) : (512 / N);
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tm + (uint32_t)((it % dslots) * N);
      for (int kb = 0; kb < 2; ++kb)
        for (int ks = 0; ks < 4; ++ks) {
          uint64_t b = sdesc(b0 + kb * 32768 + ks * 32);
          uint32_t acc = (kb | ks) != 0;
          if (kind == 0) {
            uint64_t a = sdesc(a0 + kb * 16384 + ks * 32);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                         ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
          } else {
            const uint32_t at = tm + 384 + (uint32_t)((kb * 4 + ks) * 8);   // A: 128 lanes x 8 cols per K16 step
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                         ::"r"(d), "r"(at), "l"(b), "r"(idesc), "r"(acc));
          }
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
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  struct C { int M, N, kind; } cs[] = {{128, 32, 0}, {128, 64, 0}, {128, 128, 0}, {128, 256, 0}, {128, 32, 1},
                                      {128, 64, 1}, {64, 256, 0}, {64, 128, 0}, {64, 32, 0}};
  for (auto c : cs) {
    const int iters = 2000;
    k<<<148, 128, 140000>>>(iters, c.M, c.N, c.kind, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("M %d N %d kind %d err %s\n", c.M, c.N, c.kind, cudaGetErrorString(e)); return 1; }
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s M%3d N%3d: %6.1f cycles per K16 MMA  (%.0f MAC/clk)\n", c.kind ? "TS" : "SS", c.M, c.N,
           (double)h / (iters * 8), (double)c.M * c.N * 16 / ((double)h / (iters * 8)));
  }
  return 0;
}
