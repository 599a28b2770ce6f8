// Counter-based synthetic inputs (CUDA side).  Bit-identical to spgen/gen.py;
// see that file for the recipe.  NOT product code: no method arithmetic here,
// only the input generator used by tests and bench.py to fill multi-GiB
// device buffers without a host copy.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ull;
enum { S_KNOISE = 1, S_USIGN = 2, S_QNOISE = 3, S_HEADAMP = 4, S_OUTLIER = 5, S_NEEDLE_LG = 6, S_TOKENS = 7 };
constexpr int SINK_TOKENS = 4, SINK_AMP = 96, RAMP_AMP = 32, NEEDLE_AMP = 64, OUTLIER_AMP = 200;
constexpr int QA_STRONG = 64, QA_WEAK = 16;
// "randn" mode: units of 2^-15 (the dyadic amplitudes x 512), full-mantissa bf16 (gen.py)
constexpr long long RN_UNIT = 512, RN_OUTLIER = 4LL * OUTLIER_AMP * RN_UNIT, RN_QA_OUTLIER = 160LL * RN_UNIT;
constexpr int PLANT_BASE = 40, PLANT_STEP = 4;
constexpr uint64_t VOCAB = 128256;
constexpr int MAX_SPANS = 4;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) { return mix64(seed * GOLD + stream); }
__device__ __forceinline__ uint64_t h64(uint64_t key, uint64_t idx) { return mix64(idx * GOLD + key); }
__device__ __forceinline__ long long noise4(uint64_t h) {
  return (long long)((h & 127) + ((h >> 8) & 127) + ((h >> 16) & 127) + ((h >> 24) & 127)) - 254;
}
__device__ __forceinline__ long long noise16(uint64_t h) {
  return (long long)((h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + ((h >> 48) & 0xFFFF)) - 131070;
}
__device__ __forceinline__ uint16_t rn_to_bf16_bits(long long v) {
  const float f = (float)v * 0x1p-15f;            // exact: |v| < 2^24
  const uint32_t b = __float_as_uint(f);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);   // round to nearest even
}
__device__ __forceinline__ long long usign(uint64_t key_u, long long unit, int d, int t) {
  return 1 - 2 * (long long)(h64(key_u, (uint64_t)unit * d + t) & 1);
}
__device__ __forceinline__ uint16_t to_bf16_bits(long long v) {
  float f = (float)v / 64.0f;                     // exact: |v| <= 255
  return (uint16_t)(__float_as_uint(f) >> 16);
}
__device__ __forceinline__ long long clamp255(long long v) { return v < -255 ? -255 : (v > 255 ? 255 : v); }

struct KArgs {
  uint16_t* K;
  long long k_b, k_l, k_g, k_i;       // element strides
  int B, L, Hkv, d;
  long long N_total, i0, n_local;     // global prompt length, first global token, local tokens
  uint64_t seed;
  const long long* spans;             // [B][MAX_SPANS][2] (start, end), end <= start = none
  int randn;                          // value mode: 0 dyadic, 1 full-mantissa
  const signed char* tiers;           // planted fixture: [B][n_c] chunk tiers, or null
  int chunk, pool_k;
};

__global__ void k_fill_K(KArgs a) {
  const uint64_t key_n = stream_key(a.seed, S_KNOISE), key_u = stream_key(a.seed, S_USIGN);
  const uint64_t key_o = stream_key(a.seed, S_OUTLIER), key_nlg = stream_key(a.seed, S_NEEDLE_LG);
  const long long per_row = a.d / 8;
  const long long total = (long long)a.B * a.L * a.Hkv * a.n_local * per_row;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (long long)gridDim.x * blockDim.x) {
    const int t0 = (int)(v % per_row) * 8;
    long long rest = v / per_row;
    const long long il = rest % a.n_local; rest /= a.n_local;
    const int g = (int)(rest % a.Hkv); rest /= a.Hkv;
    const int l = (int)(rest % a.L);
    const int b = (int)(rest / a.L);
    const long long i = a.i0 + il;
    const long long unit = ((long long)b * a.L + l) * a.Hkv + g;
    const bool nlg = (h64(key_nlg, (uint64_t)unit) % 10) == 0;
    bool inside = false;
    if (nlg && !a.tiers) {
      for (int s = 0; s < MAX_SPANS; ++s) {
        long long st = a.spans[(b * MAX_SPANS + s) * 2], en = a.spans[(b * MAX_SPANS + s) * 2 + 1];
        inside |= (i >= st && i < en);
      }
    }
    const long long us = a.randn ? RN_UNIT : 1;
    const long long r = (i * 64) / a.N_total;
    long long struct_amp;                          // planted boost or ramp (+ needle), times u
    if (a.tiers) {
      const long long n_c = (a.N_total + a.chunk - 1) / a.chunk;
      const long long c = i / a.chunk, j = i - c * a.chunk, hw = (a.pool_k - 1) / 2;
      const int tt = a.tiers[b * n_c + c];
      struct_amp = (tt > 0 && j >= hw && j < a.chunk - hw) ? (PLANT_BASE + PLANT_STEP * tt) * us : 0;
    } else {
      struct_amp = a.randn ? r * r * 4 : (RAMP_AMP * r * r) >> 12;
      if (inside) struct_amp += NEEDLE_AMP * us;
    }
    uint16_t out[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = t0 + j;
      const uint64_t hn = h64(key_n, ((uint64_t)unit * a.N_total + i) * a.d + t);
      const long long n = a.randn ? noise16(hn) : noise4(hn);
      const long long u = usign(key_u, unit, a.d, t);
      long long k = n;
      if (i < SINK_TOKENS) k += SINK_AMP * us * u;
      k += struct_amp * u;
      const uint64_t ho = h64(key_o, (uint64_t)unit * a.d + t);
      if (ho % 64 == 0) {
        const long long os = 1 - 2 * (long long)((ho >> 32) & 1);
        k = os * (a.randn ? RN_OUTLIER : OUTLIER_AMP) + (n >> 3);
      }
      out[j] = a.randn ? rn_to_bf16_bits(k) : to_bf16_bits(clamp255(k));
    }
    uint16_t* dst = a.K + b * a.k_b + l * a.k_l + g * a.k_g + il * a.k_i + t0;
    uint4 pk;
    pk.x = out[0] | ((uint32_t)out[1] << 16);
    pk.y = out[2] | ((uint32_t)out[3] << 16);
    pk.z = out[4] | ((uint32_t)out[5] << 16);
    pk.w = out[6] | ((uint32_t)out[7] << 16);
    *reinterpret_cast<uint4*>(dst) = pk;
  }
}

struct QArgs {
  uint16_t* Q;
  long long q_b, q_l, q_r, q_h;
  int B, L, R, H, Hkv, d;
  uint64_t seed;
  int randn;
};

__global__ void k_fill_Q(QArgs a) {
  const uint64_t key_q = stream_key(a.seed, S_QNOISE), key_u = stream_key(a.seed, S_USIGN);
  const uint64_t key_a = stream_key(a.seed, S_HEADAMP);
  const int G = a.H / a.Hkv;
  const long long total = (long long)a.B * a.L * a.R * a.H * a.d;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(v % a.d);
    long long rest = v / a.d;
    const int h = (int)(rest % a.H); rest /= a.H;
    const int r = (int)(rest % a.R); rest /= a.R;
    const int l = (int)(rest % a.L);
    const int b = (int)(rest / a.L);
    const uint64_t hq = h64(key_q, (uint64_t)v);                   // v == (((b*L+l)*R+r)*H+h)*d+t
    const long long nq = (a.randn ? noise16(hq) : noise4(hq)) >> 1;
    const long long unit = ((long long)b * a.L + l) * a.Hkv + h / G;
    const long long u = usign(key_u, unit, a.d, t);
    const uint64_t ha = h64(key_a, (uint64_t)((long long)b * a.L + l) * a.H + h);
    long long amp = (ha % 4 == 0 ? QA_STRONG : QA_WEAK) * (a.randn ? RN_UNIT : 1);
    if (a.randn && ha % 16 == 1) amp = RN_QA_OUTLIER;
    const long long q = amp * u + nq;
    a.Q[b * a.q_b + l * a.q_l + r * a.q_r + h * a.q_h + t] = a.randn ? rn_to_bf16_bits(q) : to_bf16_bits(clamp255(q));
  }
}

__global__ void k_fill_tokens(int* tok, int B, long long N, uint64_t seed) {
  const uint64_t key = stream_key(seed, S_TOKENS);
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < (long long)B * N;
       v += (long long)gridDim.x * blockDim.x)
    tok[v] = (int)(h64(key, (uint64_t)v) % VOCAB);
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g > 148 * 64 ? 148 * 64 : (g < 1 ? 1 : g));
}

}  // namespace

extern "C" {

int spgen_fill_K(void* K, long long k_b, long long k_l, long long k_g, long long k_i, int B, int L, int Hkv, int d,
                 long long N_total, long long i0, long long n_local, unsigned long long seed, const long long* spans_dev,
                 int randn, const signed char* tiers_dev, int chunk, int pool_k, void* stream) {
  if (d % 8 != 0 || (reinterpret_cast<uintptr_t>(K) & 15) != 0) return 1;
  KArgs a{reinterpret_cast<uint16_t*>(K), k_b, k_l, k_g, k_i, B, L, Hkv, d, N_total, i0, n_local, seed, spans_dev,
          randn, tiers_dev, chunk, pool_k};
  long long n = (long long)B * L * Hkv * n_local * (d / 8);
  k_fill_K<<<grid_for(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int spgen_fill_Q(void* Q, long long q_b, long long q_l, long long q_r, long long q_h, int B, int L, int R, int H, int Hkv,
                 int d, unsigned long long seed, int randn, void* stream) {
  QArgs a{reinterpret_cast<uint16_t*>(Q), q_b, q_l, q_r, q_h, B, L, R, H, Hkv, d, seed, randn};
  long long n = (long long)B * L * R * H * d;
  k_fill_Q<<<grid_for(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int spgen_fill_tokens(int* tok, int B, long long N, unsigned long long seed, void* stream) {
  k_fill_tokens<<<grid_for((long long)B * N), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(tok, B, N, seed);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // extern "C"
