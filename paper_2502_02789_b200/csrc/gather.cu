// Gather of the selected prompt tokens (merge_requests input, Alg.1):
//   out[b][j] = tokens[b][ids[b][j]]   for j < n_kept[b].   Bit-exact.
#include "sp_internal.h"

namespace sp {
namespace {

__global__ void k_gather(const int* __restrict__ tokens, const int* __restrict__ ids, const int* __restrict__ n_kept,
                         long long N, int* __restrict__ out) {
  const int b = blockIdx.y;
  const int n = n_kept[b];
  const long long base = (long long)b * N;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    out[base + j] = tokens[base + ids[base + j]];
}

}  // namespace

cudaError_t gather_launch(const int* tokens, const int* ids, const int* n_kept, int B, long long N, int* out,
                          cudaStream_t st) {
  long long blocks = (N + 255) / 256;
  if (blocks > 1184) blocks = 1184;               // 148 SMs x 8; grid-stride beyond
  dim3 grid((unsigned)blocks, (unsigned)B);
  k_gather<<<grid, 256, 0, st>>>(tokens, ids, n_kept, N, out);
  return cudaGetLastError();
}

}  // namespace sp
