// Selection: 1-D average pool -> chunk means -> top-K_c chunks -> ids/positions.
//
// PAPER.md sec:chunk_select: "we chunk the context contiguously and
// average the token score within each block, and then we select the Top-K
// blocks ... we apply a 1D average pooling before this"; sec:position_ids
// (P:125-133): kept tokens keep their original position ids.
// Readings: shrinking pool edges (Z6), partial last chunk averaged
// over its true size (Z8), K_c from the exact ppm rule (Z9, computed on the
// host), ties to the lowest chunk index (Z10), ascending ids (Z11).
//
// One CTA of 1024 threads per request.  Selection is exact and deterministic:
// a 4-pass 8-bit radix select finds the K_c-th largest chunk score (as its
// IEEE bit pattern; scores are >= 0 so bit order == value order), then an
// in-order block scan keeps every chunk above the threshold plus the
// lowest-index chunks equal to it, and compacts their token ranges.
#include "sp_internal.h"

namespace sp {
namespace {

constexpr int ST = 1024;
constexpr int NW = ST / 32;

struct ScanSmem {
  int warp_tot[NW];
  int total;
};

// Block-wide exclusive scan of v (all ST threads participate); returns the
// exclusive prefix, writes the block total to *total.
__device__ __forceinline__ int block_excl_scan(int v, ScanSmem& sm, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int t = lane < NW ? sm.warp_tot[lane] : 0;
    int u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += y;
    }
    if (lane < NW) sm.warp_tot[lane] = u - t;    // exclusive warp offsets
    if (lane == 31) sm.total = u;
  }
  __syncthreads();
  int res = sm.warp_tot[warp] + x - v;
  *total = sm.total;
  __syncthreads();                                 // sm reusable after return
  return res;
}

__global__ void __launch_bounds__(ST) k_select(const float* __restrict__ imp_all, long long N, int pool_k, int chunk,
                                               int pos0, long long K_c, int* __restrict__ ids_all,
                                               int* __restrict__ pos_all, int* __restrict__ n_kept,
                                               float* __restrict__ cs_all) {
  __shared__ float tile[ST];
  __shared__ unsigned hist[256];
  __shared__ unsigned s_digit, s_remaining;
  __shared__ ScanSmem scan;
  const int b = blockIdx.x, tid = threadIdx.x;
  const long long n_c = (N + chunk - 1) / chunk;
  const float* imp = imp_all + (long long)b * N;
  float* cs = cs_all + (long long)b * n_c;
  int* ids = ids_all + (long long)b * N;
  int* pos = pos_all + (long long)b * N;
  const long long w = (pool_k - 1) / 2;

  // ---- A. pooled scores (centred window, shrinking edges) -> chunk sums, in token order
  for (long long base = 0; base < N; base += ST) {
    const long long i = base + tid;
    if (i < N) {
      long long lo = i - w < 0 ? 0 : i - w, hi = i + w > N - 1 ? N - 1 : i + w;
      float s = 0.f;
      for (long long j = lo; j <= hi; ++j) s += imp[j];
      tile[tid] = s / (float)(hi - lo + 1);
    }
    __syncthreads();
    const long long tend = (base + ST < N) ? base + ST : N;
    const long long c_first = base / chunk, c_last = (tend - 1) / chunk;
    for (long long c = c_first + tid; c <= c_last; c += ST) {
      long long t0 = c * chunk > base ? c * chunk : base;
      long long t1 = (c + 1) * chunk < tend ? (c + 1) * chunk : tend;
      float s = (t0 == c * chunk) ? 0.f : cs[c];      // chunk continued from the previous tile
      for (long long t = t0; t < t1; ++t) s += tile[t - base];
      cs[c] = s;
    }
    __syncthreads();
  }
  for (long long c = tid; c < n_c; c += ST) {
    long long sz = ((c + 1) * chunk < N ? (c + 1) * chunk : N) - c * chunk;
    cs[c] = cs[c] / (float)sz;
  }
  __syncthreads();

  // ---- B. radix select: threshold bit pattern T of the K_c-th largest score
  unsigned prefix = 0, pmask = 0;
  unsigned remaining = (unsigned)K_c;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int k = tid; k < 256; k += ST) hist[k] = 0;
    __syncthreads();
    for (long long c = tid; c < n_c; c += ST) {
      unsigned key = __float_as_uint(cs[c]);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      unsigned cum = 0, dgt = 0;
      for (int k = 255; k >= 0; --k) {
        if (cum + hist[k] >= remaining) { dgt = (unsigned)k; break; }
        cum += hist[k];
      }
      s_digit = dgt;
      s_remaining = remaining - cum;
    }
    __syncthreads();
    prefix |= s_digit << shift;
    pmask |= 255u << shift;
    remaining = s_remaining;
    __syncthreads();
  }
  const unsigned T = prefix;
  const int need_eq = (int)remaining;            // chunks equal to T to keep (lowest indices first)

  // ---- C. keep flags in chunk order, compaction of the kept token ranges
  int carry_eq = 0, carry_tok = 0;
  for (long long base = 0; base < n_c; base += ST) {
    const long long c = base + tid;
    unsigned key = c < n_c ? __float_as_uint(cs[c]) : 0u;
    int eq = (c < n_c && key == T) ? 1 : 0;
    int gt = (c < n_c && key > T) ? 1 : 0;
    int tot;
    int eq_rank = block_excl_scan(eq, scan, &tot) + carry_eq;
    carry_eq += tot;
    int keep = gt | (eq & (eq_rank < need_eq ? 1 : 0));
    int sz = 0;
    if (keep) sz = (int)(((c + 1) * chunk < N ? (c + 1) * chunk : N) - c * chunk);
    int off = block_excl_scan(sz, scan, &tot) + carry_tok;
    carry_tok += tot;
    if (keep) {
      const int t0 = (int)(c * chunk);
      for (int j = 0; j < sz; ++j) {
        ids[off + j] = t0 + j;
        pos[off + j] = t0 + j + pos0;
      }
    }
  }
  if (tid == 0) n_kept[b] = carry_tok;
}

}  // namespace

size_t select_ws_bytes(int B, long long N, int chunk) {
  long long n_c = (N + chunk - 1) / chunk;
  return align256((size_t)B * n_c * sizeof(float));
}

cudaError_t select_launch(const float* imp, int B, long long N, int pool_k, int chunk, int pos0, long long K_c,
                          int* ids, int* pos, int* n_kept, void* ws, cudaStream_t st) {
  k_select<<<B, ST, 0, st>>>(imp, N, pool_k, chunk, pos0, K_c, ids, pos, n_kept, reinterpret_cast<float*>(ws));
  return cudaGetLastError();
}

}  // namespace sp
