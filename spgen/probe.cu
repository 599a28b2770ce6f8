// HBM read-stream probes for bench.py's second roofline denominator (SURVEY
// 8(d): "a read-only stream peak the bench measures itself").  NOT product
// code and no method arithmetic: two ways of reading a large device buffer
// once, as fast as the memory system allows.
//   mode 0: 1-D cp.async.bulk (TMA) of 32 KiB tiles into a 6-stage SMEM ring per
//           CTA, one CTA per SM (the score kernel's way of reading K);
//   mode 1: 128-bit ld.global.nc, 8 loads in flight per thread, xor-reduced
//           into one word per CTA (the "vectorized read-reduce").
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int kTile = 32768, kStages = 6;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) k_read_tma(const uint8_t* src, long long tiles, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(buf + kStages * kTile);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2 * kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long per = (tiles + gridDim.x - 1) / gridDim.x;
  const long long t0 = blockIdx.x * per, t1 = t0 + per < tiles ? t0 + per : tiles;
  if (threadIdx.x == 0) {                                   // producer
    int st = 0; uint32_t ph = 0;
    for (long long t = t0; t < t1; ++t) {
      asm volatile("{\n.reg .pred p;\nW0: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W0;\n}"
                   ::"r"(smem_u32(bars + kStages + st)), "r"(ph ^ 1) : "memory");
      const uint32_t full = smem_u32(bars + st);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(kTile) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf + st * kTile)), "l"(src + t * kTile), "r"(kTile), "r"(full) : "memory");
      if (++st == kStages) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {                           // consumer: frees each stage once it landed
    int st = 0; uint32_t ph = 0;
    unsigned x = 0;
    for (long long t = t0; t < t1; ++t) {
      asm volatile("{\n.reg .pred p;\nW1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}"
                   ::"r"(smem_u32(bars + st)), "r"(ph) : "memory");
      x ^= *reinterpret_cast<const unsigned*>(buf + st * kTile);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + kStages + st)) : "memory");
      if (++st == kStages) { st = 0; ph ^= 1; }
    }
    if (x == 0x12345678u) *sink = x;                        // keep the reads observable
  }
}

__global__ void __launch_bounds__(512) k_read_ld(const uint4* __restrict__ src, long long n16, unsigned* sink) {
  unsigned x = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) x ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  for (; i < n16; i += stride) {
    const uint4 v = __ldg(src + i);
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x12345678u) *sink = x;
}

}  // namespace

extern "C" int spgen_read_stream(const void* buf, long long bytes, int mode, void* sink, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (mode == 0) {
    const size_t smem = kStages * kTile + 2 * kStages * 8 + 1024;
    if (cudaFuncSetAttribute(k_read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return 2;
    k_read_tma<<<sms, 64, smem, st>>>(reinterpret_cast<const uint8_t*>(buf), bytes / kTile,
                                      reinterpret_cast<unsigned*>(sink));
  } else {
    k_read_ld<<<sms * 4, 512, 0, st>>>(reinterpret_cast<const uint4*>(buf), bytes / 16,
                                        reinterpret_cast<unsigned*>(sink));
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
