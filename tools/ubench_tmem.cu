// Microbenchmark: tcgen05.ld (TMEM -> registers) latency / throughput on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tmem tools/ubench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int NB>
__global__ void k(int iters, int nwarps_active, unsigned long long* out, float* sink) {
  __shared__ uint32_t base_s;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&base_s)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = base_s;
  float acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.f;
  unsigned long long t0 = clock64();
  if (warp < nwarps_active) {
    const uint32_t lanebase = tm + ((uint32_t)((warp & 3) * 32) << 16);
    for (int i = 0; i < iters; ++i) {
      uint32_t r[NB][32];
#pragma unroll
      for (int j = 0; j < NB; ++j) ld32(lanebase + ((i * NB + j) * 32) % 512, r[j]);
      wait_ld();
#pragma unroll
      for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] += __uint_as_float(r[j][c]);
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x % 32 == 0 && blockIdx.x == 0) out[warp] = t1 - t0;
  float tot = 0.f;
#pragma unroll
  for (int c = 0; c < 32; ++c) tot += acc[c];
  if (tot == 1.2345f) sink[threadIdx.x] = tot;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 64 * 8);
  cudaMalloc(&sink, 4096);
  unsigned long long h[16];
  const int iters = 2000;
  for (int nw : {1, 4, 8, 16}) {
    for (int nb : {1, 2, 4}) {
      int threads = 32 * (nw < 4 ? 4 : nw);
      if (nb == 1) k<1><<<148, threads>>>(iters, nw, d, sink);
      if (nb == 2) k<2><<<148, threads>>>(iters, nw, d, sink);
      if (nb == 4) k<4><<<148, threads>>>(iters, nw, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
      double cyc = (double)h[0] / (iters);
      double bytes_per_cyc = (double)nw * nb * 32 * 32 * 4 / cyc;
      printf("warps %2d batch %d : %.1f cycles per batch (warp0), %.1f B/cycle/SM\n", nw, nb, cyc, bytes_per_cyc);
    }
  }
  return 0;
}
