// SIMT (FP32 FMA) two-pass token-importance kernels.
//
// This is the baseline the fused tcgen05 kernel (score_fused.cu) is measured
// against, and the compute behind the sequence-sharded split API
// (sp_score_stats / sp_score_finish).  It reads K twice (pass 1: softmax
// statistics, pass 2: the (l,h)-max), so it is bounded by 50% of the HBM
// roofline before the FMA-rate limit.
//
// Math (O1-O4; PAPER.md sec:token_importance P:105-107, sec:attn_agg P:119):
//   x[l,h,r,i]  = scale*log2(e) * <Q[l][r][h], K[l][h/G][i]>       (log2-domain logit)
//   lse2[l,h,r] = log2 sum_i 2^x                                   (softmax over the prompt, Z2)
//   acc[r,i]    = max_{l,h} (x - lse2)                              (max over H and L)
//   imp[i]      = (1/Rv) sum_r 2^acc[r,i]                           (mean over valid rows)
#include "sp_internal.h"

#include <math_constants.h>

namespace sp {
namespace {

constexpr int TB = 128;    // tokens per CTA (one per thread)
constexpr int CB = 32;     // logit columns per pass

__device__ __forceinline__ void set_err(int* err, int code) { atomicCAS(err, 0, code); }

// Load the unit's Q columns [c0, c0+CB) into shared memory as fp32.
// Column c = r*G + hh  (row r of the look-ahead, query head g*G + hh).
__device__ void load_q_cols(const __nv_bfloat16* Q, const Geom& g, const Layout& lay, int b, int l, int kv,
                            int c0, int ncols, float* qs) {
  for (int e = threadIdx.x; e < CB * g.d; e += blockDim.x) {
    int c = e / g.d, t = e % g.d;
    float v = 0.f;
    if (c < ncols) {
      int col = c0 + c, r = col / g.G, hh = col % g.G;
      const __nv_bfloat16* q = Q + b * lay.q_b + l * lay.q_l + r * lay.q_r + (long long)(kv * g.G + hh) * lay.q_h;
      v = __bfloat162float(q[t]);
    }
    qs[c * g.d + t] = v;
  }
}

// acc[c] = <Q col c, K row> for CB columns; K row is d contiguous bf16.
__device__ __forceinline__ void dot_cols(const __nv_bfloat16* krow, int d, const float* qs, float (&acc)[CB]) {
#pragma unroll
  for (int c = 0; c < CB; ++c) acc[c] = 0.f;
  for (int t0 = 0; t0 < d; t0 += 8) {
    uint4 raw = *reinterpret_cast<const uint4*>(krow + t0);
    const __nv_bfloat162* kp = reinterpret_cast<const __nv_bfloat162*>(&raw);
    float kf[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(kp[j]);
      kf[2 * j] = f.x; kf[2 * j + 1] = f.y;
    }
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const float4* qv = reinterpret_cast<const float4*>(qs + c * d + t0);
      float4 a = qv[0], b2 = qv[1];
      float s = acc[c];
      s = fmaf(kf[0], a.x, s); s = fmaf(kf[1], a.y, s); s = fmaf(kf[2], a.z, s); s = fmaf(kf[3], a.w, s);
      s = fmaf(kf[4], b2.x, s); s = fmaf(kf[5], b2.y, s); s = fmaf(kf[6], b2.z, s); s = fmaf(kf[7], b2.w, s);
      acc[c] = s;
    }
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Pass 1: per (unit, token block) partial statistics (m2, l) for every column.
// part[row][tb][2], row = ((b*L + l)*H + h)*Rv + r.  Also initialises acc (-inf)
// for the block's tokens when l == 0 && kv == 0 (acc != nullptr).
__global__ void __launch_bounds__(TB) k_stats(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                                              Geom g, Layout lay, float* __restrict__ part, int ntb,
                                              unsigned* __restrict__ acc) {
  extern __shared__ float qs[];                 // [CB][d]
  __shared__ float red[TB / 32][CB];
  __shared__ float mcol[CB];
  const int unit = blockIdx.y;                  // (b*L + l)*Hkv + kv
  const int kv = unit % g.Hkv, l = (unit / g.Hkv) % g.L, b = unit / (g.Hkv * g.L);
  const int tb = blockIdx.x;
  const long long i = (long long)tb * TB + threadIdx.x;
  const bool valid = i < g.N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float xs = g.scale * kLog2e;
  if (acc != nullptr && l == 0 && kv == 0 && valid)
    for (int r = 0; r < g.Rv; ++r) acc[((long long)b * g.Rv + r) * g.N + i] = 0xFF800000u;   // -inf
  const __nv_bfloat16* krow = K + b * lay.k_b + l * lay.k_l + kv * lay.k_g + (valid ? i : 0) * lay.k_i;
  const int ncol = g.G * g.Rv;
  for (int c0 = 0; c0 < ncol; c0 += CB) {
    __syncthreads();
    load_q_cols(Q, g, lay, b, l, kv, c0, min(CB, ncol - c0), qs);
    __syncthreads();
    float x[CB];
    dot_cols(krow, g.d, qs, x);
#pragma unroll
    for (int c = 0; c < CB; ++c) x[c] = valid ? x[c] * xs : -CUDART_INF_F;
    // column max over the block
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      float m = warp_max(x[c]);
      if (lane == 0) red[warp][c] = m;
    }
    __syncthreads();
    if (threadIdx.x < CB) {
      float m = red[0][threadIdx.x];
      for (int w = 1; w < TB / 32; ++w) m = fmaxf(m, red[w][threadIdx.x]);
      mcol[threadIdx.x] = m;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      float e = valid ? exp2f(x[c] - mcol[c]) : 0.f;
      float s = warp_sum(e);
      if (lane == 0) red[warp][c] = s;
    }
    __syncthreads();
    if (threadIdx.x < CB && c0 + threadIdx.x < ncol) {
      float s = 0.f;
      for (int w = 0; w < TB / 32; ++w) s += red[w][threadIdx.x];
      int col = c0 + threadIdx.x, r = col / g.G, hh = col % g.G;
      long long row = (((long long)b * g.L + l) * g.H + kv * g.G + hh) * g.Rv + r;
      part[(row * ntb + tb) * 2 + 0] = mcol[threadIdx.x];
      part[(row * ntb + tb) * 2 + 1] = s;
    }
  }
}

// Merge partial statistics in part order (deterministic).
// mode 0: part is [rows][nparts][2] (per token block), out[row] = lse2 = m + log2(l)
// mode 1: part is [rows][nparts][2],                    out[row][2] = (m, l)
// mode 2: part is [nparts][rows][2] (per rank),          out[row] = lse2
__global__ void k_combine(const float* __restrict__ part, int nparts, long long rows, float* __restrict__ out,
                          int mode, int* err) {
  long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  auto idx = [&](int p) -> long long { return mode == 2 ? (long long)p * rows + row : row * nparts + p; };
  float m = -CUDART_INF_F;
  for (int p = 0; p < nparts; ++p) m = fmaxf(m, part[idx(p) * 2]);
  float s = 0.f;
  for (int p = 0; p < nparts; ++p) {
    float mp = part[idx(p) * 2], lp = part[idx(p) * 2 + 1];
    if (lp > 0.f) s += lp * exp2f(mp - m);
  }
  if (mode == 1) {
    out[row * 2] = m;
    out[row * 2 + 1] = s;
  } else {
    float lse2 = m + log2f(s);
    if (!isfinite(lse2)) set_err(err, kDevNonFinite);
    out[row] = lse2;
  }
}

// Pass 2: acc[b][r][i] = max over (l, h) of (x - lse2), via atomicMin on the bit
// pattern of non-positive floats (order-independent, hence deterministic).
__global__ void __launch_bounds__(TB) k_finish(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                                               Geom g, Layout lay, const float* __restrict__ lse2,
                                               unsigned* __restrict__ acc) {
  extern __shared__ float qs[];
  __shared__ float ls[CB];
  const int unit = blockIdx.y;
  const int kv = unit % g.Hkv, l = (unit / g.Hkv) % g.L, b = unit / (g.Hkv * g.L);
  const long long i = (long long)blockIdx.x * TB + threadIdx.x;
  const bool valid = i < g.N;
  const float xs = g.scale * kLog2e;
  const __nv_bfloat16* krow = K + b * lay.k_b + l * lay.k_l + kv * lay.k_g + (valid ? i : 0) * lay.k_i;
  const int ncol = g.G * g.Rv;
  for (int c0 = 0; c0 < ncol; c0 += CB) {
    __syncthreads();
    load_q_cols(Q, g, lay, b, l, kv, c0, min(CB, ncol - c0), qs);
    if (threadIdx.x < CB) {
      int col = c0 + threadIdx.x;
      float v = CUDART_INF_F;
      if (col < ncol) {
        int r = col / g.G, hh = col % g.G;
        v = lse2[(((long long)b * g.L + l) * g.H + kv * g.G + hh) * g.Rv + r];
      }
      ls[threadIdx.x] = v;
    }
    __syncthreads();
    float x[CB];
    dot_cols(krow, g.d, qs, x);
    if (!valid) continue;
    // columns are r-major: c = r*G + hh; take the max over hh for each r and
    // fold it into acc (a row's columns may straddle two column blocks: the
    // max of the two partial maxima is the same max)
    const int nc = min(CB, ncol - c0);
    int cur_r = c0 / g.G;
    float best = -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      if (c < nc) {
        int r = (c0 + c) / g.G;
        if (r != cur_r) {
          atomicMin(&acc[((long long)b * g.Rv + cur_r) * g.N + i], __float_as_uint(fminf(best, -0.0f)));
          best = -CUDART_INF_F;
          cur_r = r;
        }
        best = fmaxf(best, x[c] * xs - ls[c]);
      }
    }
    atomicMin(&acc[((long long)b * g.Rv + cur_r) * g.N + i], __float_as_uint(fminf(best, -0.0f)));
  }
}

__global__ void k_importance(const unsigned* __restrict__ acc, Geom g, float* __restrict__ imp) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int b = blockIdx.y;
  if (i >= g.N) return;
  float s = 0.f;
  for (int r = 0; r < g.Rv; ++r) s += exp2f(__uint_as_float(acc[((long long)b * g.Rv + r) * g.N + i]));
  imp[(long long)b * g.N + i] = s / (float)g.Rv;
}

// dynamic loops in dot_cols index registers with a runtime d; keep d%8==0
size_t qs_bytes(const Geom& g) { return (size_t)CB * g.d * sizeof(float); }
long long n_tb(const Geom& g) { return (g.N + TB - 1) / TB; }
long long n_rows(const Geom& g) { return (long long)g.B * g.L * g.H * g.Rv; }

}  // namespace

size_t simt_split_ws_bytes(const Geom& g) {
  return align256((size_t)n_rows(g) * n_tb(g) * 2 * sizeof(float));
}

size_t simt_score_ws_bytes(const Geom& g) {
  return simt_split_ws_bytes(g) + align256((size_t)n_rows(g) * sizeof(float)) +
         align256((size_t)g.B * g.Rv * g.N * sizeof(unsigned));
}

cudaError_t simt_score_stats(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                             float* stats, void* ws, cudaStream_t st) {
  float* part = reinterpret_cast<float*>(ws);
  dim3 grid((unsigned)n_tb(g), (unsigned)(g.B * g.L * g.Hkv));
  k_stats<<<grid, TB, qs_bytes(g), st>>>(Q, K, g, lay, part, (int)n_tb(g), nullptr);
  long long rows = n_rows(g);
  k_combine<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(part, (int)n_tb(g), rows, stats, 1,
                                                            device_error_flag());
  return cudaGetLastError();
}

cudaError_t stats_combine(const float* parts, int P, long long rows, float* lse2, cudaStream_t st) {
  k_combine<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(parts, P, rows, lse2, 2 /*rank-major*/,
                                                            device_error_flag());
  return cudaGetLastError();
}

cudaError_t simt_score_finish(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                              const float* lse2, float* importance, void* ws, cudaStream_t st) {
  unsigned* acc = reinterpret_cast<unsigned*>(ws);
  long long nacc = (long long)g.B * g.Rv * g.N;
  cudaError_t e = cudaMemsetAsync(acc, 0xFF, nacc * sizeof(unsigned), st);   // 0xFFFFFFFF > any -x bits
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)n_tb(g), (unsigned)(g.B * g.L * g.Hkv));
  k_finish<<<grid, TB, qs_bytes(g), st>>>(Q, K, g, lay, lse2, acc);
  dim3 g2((unsigned)((g.N + 255) / 256), (unsigned)g.B);
  k_importance<<<g2, 256, 0, st>>>(acc, g, importance);
  return cudaGetLastError();
}

cudaError_t simt_score(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                       float* importance, void* ws, cudaStream_t st) {
  char* p = reinterpret_cast<char*>(ws);
  float* part = reinterpret_cast<float*>(p);
  p += simt_split_ws_bytes(g);
  float* lse2 = reinterpret_cast<float*>(p);
  p += align256((size_t)n_rows(g) * sizeof(float));
  unsigned* acc = reinterpret_cast<unsigned*>(p);
  dim3 grid((unsigned)n_tb(g), (unsigned)(g.B * g.L * g.Hkv));
  k_stats<<<grid, TB, qs_bytes(g), st>>>(Q, K, g, lay, part, (int)n_tb(g), acc);
  long long rows = n_rows(g);
  k_combine<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(part, (int)n_tb(g), rows, lse2, 0,
                                                            device_error_flag());
  k_finish<<<grid, TB, qs_bytes(g), st>>>(Q, K, g, lay, lse2, acc);
  dim3 g2((unsigned)((g.N + 255) / 256), (unsigned)g.B);
  k_importance<<<g2, 256, 0, st>>>(acc, g, importance);
  return cudaGetLastError();
}

}  // namespace sp
