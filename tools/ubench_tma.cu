// Microbenchmark: HBM read bandwidth of TMA streaming into SMEM on sm_100a.
//  mode 0: 2-D tensor map [rows][128] bf16, SWIZZLE_128B, box {64,128} x2 per 32 KiB stage (as the fused kernel)
//  mode 1: 1-D cp.async.bulk of 32 KiB contiguous per stage
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma tools/ubench_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void arrive(uint32_t bar) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory"); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(bar), "r"(par) : "memory");
}

__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap map, const uint8_t* src, long long tiles_per_cta,
                                           int stages, int mode, int reread) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(buf + stages * 32768);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(smem_u32(bars + s), 1); mbar_init(smem_u32(bars + stages + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long t0 = blockIdx.x * tiles_per_cta;
  if (warp == 0 && threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    const long long total = reread > 0 ? 2 * tiles_per_cta : tiles_per_cta;
    for (long long it = 0; it < total; ++it) {
      // reread > 0: every other load re-reads the tile `reread` tiles back (L2 hit if still resident)
      long long t = reread > 0 ? it / 2 : it;
      if (reread > 0 && (it & 1)) t = t - reread < 0 ? t : t - reread;
      wait(smem_u32(bars + stages + st), ph ^ 1);
      const uint32_t full = smem_u32(bars + st);
      expect_tx(full, 32768);
      const uint32_t dst = smem_u32(buf + st * 32768);
      const long long row = (t0 + t) * 128;
      if (mode == 0) {
        for (int kb = 0; kb < 2; ++kb)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                       ::"r"(dst + kb * 16384), "l"((uint64_t)&map), "r"(full), "r"(kb * 64), "r"((int)row) : "memory");
      } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src + row * 256), "r"(32768), "r"(full) : "memory");
      }
      if (++st == stages) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    const long long total = reread > 0 ? 2 * tiles_per_cta : tiles_per_cta;
    for (long long t = 0; t < total; ++t) {
      wait(smem_u32(bars + st), ph);
      arrive(smem_u32(bars + stages + st));
      if (++st == stages) { st = 0; ph ^= 1; }
    }
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const long long bytes = 2LL << 30, rows = bytes / 256;
  uint8_t* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows}, strides[1] = {256};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  for (int prom = 0; prom < 1; ++prom) {
    CUtensorMapL2promotion pr = prom == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : prom == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    ((Enc)fp)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int reread : {0, 8, 32, 64}) {
    for (int mode = 0; mode < 1; ++mode) {
      for (int stages : {4, 6}) {
        const int ctas = 148;
        const long long tpc = rows / 128 / ctas;
        size_t smem = stages * 32768 + 2048;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        k<<<ctas, 64, smem>>>(map, d, tpc, stages, mode, reread);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k<<<ctas, 64, smem>>>(map, d, tpc, stages, mode, reread);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double gbs = 5.0 * tpc * ctas * 32768 / (ms / 1000.0) / 1e9;
        printf("reread %d stages %d: HBM-equivalent %.0f GB/s (SMEM fill %.0f GB/s)\n", reread, stages, gbs,
               gbs * (reread > 0 ? 2 : 1));
      }
    }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
