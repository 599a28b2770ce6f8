// Selection: 1-D average pool -> chunk means -> top-K_c chunks -> ids/positions
// (+ optionally the token gather), and its sequence-sharded split into a
// rank-local candidate select and a global candidate merge.
//
// PAPER.md sec:chunk_select: "we chunk the context contiguously and
// average the token score within each block, and then we select the Top-K
// blocks ... we apply a 1D average pooling before this"; sec:position_ids
// (P:125-133): kept tokens keep their original position ids; Alg.1
// merge_requests takes the selected tokens.  Under the paper's TP=8 placement
// the prompt is split along tokens.
// Readings: shrinking pool edges (Z6), partial last chunk averaged
// over its true size (Z8), K_c from the exact ppm rule (Z9, computed on the
// host), ties to the lowest chunk index (Z10), ascending ids (Z11).
//
// One launch.  Phase A can run on many CTAs per request (kModeA: grid (B, chunk
// blocks), writing cs to the workspace), the request's last CTA to finish it
// continuing with phases B-C (1024 threads); short prompts run all three on one
// CTA per request (kModeAll).  Launched as a programmatic dependent of the
// score kernel (its prologue overlaps the score kernel's tail):
//   A. importance is staged in shared memory segment by segment (all loads of a
//      segment in flight together), pooled, and summed per chunk (a canonical
//      order that depends only on the chunk: segments are chunk-aligned, so the
//      single-GPU, multi-CTA and sequence-sharded runs give the same bits);
//   B. a 4-pass 8-bit radix select on the IEEE bits of cs (scores are >= 0, so
//      bit order == value order) finds the K-th largest value T; the digit
//      search is a parallel suffix scan over the 256 bins;
//   C. an in-order block scan keeps every chunk above T plus the lowest-index
//      chunks equal to T (exactly K chunks), compacts their token ranges into
//      ids/pos -- one warp per kept chunk, coalesced -- and, if requested,
//      gathers the kept tokens in the same pass.
// Variants (template parameter V):
//   kPlain -- the whole prompt on one GPU (sp_select, sp_select_gather, ragged);
//   kCand  -- sequence shard: phase A over this rank's chunks (pooling windows
//             reach into the neighbours' importance through the exchanged edge
//             values), B-C with K = M = min(K_c, n_c / P), and the kept chunks
//             written as 64-bit candidate keys (score bits << 32 | ~chunk): as
//             unsigned integers they order exactly as (score desc, index asc);
//   kMerge -- the P ranks' gathered candidates scattered into the dense chunk
//             array (absent chunks marked invalid), B-C with K = K_c over the
//             whole prompt: the global top-K_c is a subset of the union of the
//             local top-M lists because every rank ranks by the same total order.
#include "select_body.cuh"

#include <algorithm>
#include <cstdlib>

namespace sp {
namespace {

using namespace sel;
constexpr int ST = 1024;

}  // namespace
#ifdef SP_SELECT_TRACE
// [0] first CTA entry, [1] first CTA past griddepcontrol.wait, [2] phase A done
// (last CTA), [3] B-C start, [4] B done, [5] C done
extern "C" int sp_select_trace_read(unsigned long long* host8, int reset) {   // 16 stamps
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(host8, sel::g_sel_trace, sizeof(g_sel_trace)) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long init[16] = {~0ull, ~0ull};
    if (cudaMemcpyToSymbol(sel::g_sel_trace, init, sizeof(init)) != cudaSuccess) return 1;
  }
  return 0;
}
#endif
namespace {

template <int V>
__global__ void __launch_bounds__(ST) k_select(SelArgs a) {
  extern __shared__ __align__(16) float dyn[];    // [segcap + 2w] staged importance, [segcap] pooled, [n_c] scores
  SEL_STAMP_MIN(0);
  // programmatic dependent launch: this grid may start while the producer of
  // the importance (the score kernel) is finishing; wait for its results here,
  // then let the next dependent launch begin its own prologue
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  SEL_STAMP_MIN(1);
  SelShared<ST>& sh = *reinterpret_cast<SelShared<ST>*>(dyn + a.sh_off);
  select_body<V, ST>(a, blockIdx.x, blockIdx.y, dyn, sh);
}

__global__ void k_seq_edges(const float* __restrict__ imp, long long n, int w, float* __restrict__ edges) {
  const int b = blockIdx.x;
  for (int j = threadIdx.x; j < 2 * w; j += blockDim.x)
    edges[(long long)b * 2 * w + j] = imp[(long long)b * n + (j < w ? j : n - 2 * w + j)];
}

constexpr size_t kSmemMax = (size_t)(2 * SEG + 2 * ((kMaxPool - 1) / 2) + kSmemChunks + 4) * sizeof(float) +
                            sizeof(SelShared<ST>);

// The >48 KiB dynamic-SMEM opt-in is a per-device function attribute: set it
// once per (device, variant).
template <int V>
cudaError_t configure() {
  static bool done[64][1] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!done[dev][0]) {
    e = cudaFuncSetAttribute(k_select<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
    if (e != cudaSuccess) return e;
    done[dev][0] = true;
  }
  return cudaSuccess;
}

// Development A/B knobs (timing only): SP_SELECT_NO_PDL=1 launches without the
// programmatic-dependent attribute.
bool select_pdl() {
  static const bool on = std::getenv("SP_SELECT_NO_PDL") == nullptr;
  return on;
}

template <int V>
cudaError_t launch_pdl(dim3 grid, size_t smem, cudaStream_t st, const SelArgs& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(ST);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlap with the producer's tail
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = select_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_select<V>, a);
}

// Long ranges: phase A over `nblk` blocks of cpb chunks of each request
// (kModeA), the last block of a request continuing with B-C; one kModeAll CTA
// per request otherwise.  Either way one launch.
template <int V>
cudaError_t launch_select(SelArgs a, int B, long long n_tok, long long n_chunks, cudaStream_t st) {
  cudaError_t e = configure<V>();
  if (e != cudaSuccess) return e;
  const long long w = (a.pool_k - 1) / 2;
  const int chunk = a.chunk;
  static const long long kTokPerCta = std::getenv("SP_SELECT_TPC") ? std::atoll(std::getenv("SP_SELECT_TPC")) : 2048;
  const long long cpb = std::max(1LL, kTokPerCta / chunk);
  const long long nblk = (n_chunks + cpb - 1) / cpb;
  const long long cs_floats = n_chunks <= kSmemChunks ? n_chunks : 0;
  a.nreq = B;
  auto smem_for = [&](int segcap) {                 // staged region (16-byte aligned), then the scratch
    a.sh_off = (int)((2 * segcap + 2 * w + cs_floats + 3) / 4 * 4);
    return (size_t)a.sh_off * sizeof(float) + sizeof(SelShared<ST>);
  };
  if (V != kMerge && nblk >= 4 && nblk <= 65535) {
    const long long span = std::min(n_tok, cpb * chunk);
    a.segcap = chunk > SEG ? SEG : (int)std::min<long long>(SEG, (span + 31) / 32 * 32);
    a.cpb = cpb;
    a.nblk = (int)nblk;
    a.mode = kModeA;
    const size_t smem = smem_for(a.segcap);
    return launch_pdl<V>(dim3(B, (unsigned)nblk), smem, st, a);
  }
  a.segcap = SEG;
  a.cpb = n_chunks;
  a.nblk = 1;
  a.mode = kModeAll;
  const size_t smem = smem_for(SEG);
  return launch_pdl<V>(dim3(B), smem, st, a);
}

}  // namespace

// [B] phase-A completion counters (zero-filled once, self-resetting; first, so
// their place does not depend on N or chunk), then [B][n_c] chunk scores
size_t select_ws_bytes(int B, long long N, int chunk) {
  long long n_c = (N + chunk - 1) / chunk;
  return align256((size_t)B * sizeof(unsigned)) + align256((size_t)B * n_c * sizeof(float));
}

namespace {
unsigned* ws_counters(void* ws) { return reinterpret_cast<unsigned*>(ws); }
float* ws_scores(void* ws, int B) {
  return reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align256((size_t)B * sizeof(unsigned)));
}
}  // namespace

float* select_ws_scores(void* ws, int B) { return ws_scores(ws, B); }

// Deferred finalize (sp_score_select): phase A over CTAs of about 8 * NT /
// (n_ug * Rv) tokens (8 partial-map loads per thread), computing the importance from the score
// kernel's partial maps, writing it, then the usual pooling and chunk means;
// the request's last CTA runs B-C.
namespace {
// launch shape of the deferred-finalize selection; false: not supported
// tokens per CTA: about 8 partial-map loads per thread, one batch in flight (A/B
// SP_DEFER_LOADS: 8 beat 16 by 0.4-0.8 us per step at C1-C3; 4 needs two waves of CTAs at C3)
bool deferred_shape(SelArgs& a, long long N, int Rv, int n_ug, int pool_k, int chunk, long long* nblk_out,
                    size_t* smem_out) {
  const long long n_c = (N + chunk - 1) / chunk;
  const long long w = (pool_k - 1) / 2;
  static const long long loads = std::getenv("SP_DEFER_LOADS") ? std::atoll(std::getenv("SP_DEFER_LOADS")) : 8;
  const long long want = std::max<long long>(32, (loads * ST) / std::max(1, n_ug * Rv));
  const long long tok = std::max<long long>(chunk, std::min<long long>(2048, want) / chunk * chunk);
  const long long cpb = std::max(1LL, tok / chunk);
  const long long nblk = (n_c + cpb - 1) / cpb;
  if (nblk > 65535 || cpb * chunk > SEG || pool_k > kMaxPool) return false;
  a.segcap = (int)std::min<long long>(SEG, (std::min(N, cpb * chunk) + 31) / 32 * 32);
  a.cpb = cpb;
  a.nblk = (int)nblk;
  a.mode = kModeA;
  const long long cs_floats = n_c <= kSmemChunks ? n_c : 0;
  const long long staged = 2 * a.segcap + 2 * w + cs_floats;
  a.mb_off = (int)((staged + 3) / 4 * 4);
  const long long mb = (long long)Rv * (a.segcap + 2 * w);
  a.sh_off = (int)((a.mb_off + mb + 3) / 4 * 4);
  *nblk_out = nblk;
  *smem_out = (size_t)a.sh_off * sizeof(float) + sizeof(SelShared<ST>);
  return *smem_out <= kSmemMax;
}
}  // namespace

bool select_deferred_supported(long long N, int Rv, int n_ug, int pool_k, int chunk) {
  SelArgs a{};
  long long nblk;
  size_t smem;
  return deferred_shape(a, N, Rv, n_ug, pool_k, chunk, &nblk, &smem);
}

cudaError_t select_deferred_launch(const float* accp, long long pitch, int n_ug, int Rv, float* imp_out, int B, long long N,
                                   int pool_k, int chunk, int pos0, long long ppm, int* ids, int* pos, int* n_kept,
                                   void* ws, cudaStream_t st, const int* tokens, int* out) {
  cudaError_t e = configure<kPlain>();
  if (e != cudaSuccess) return e;
  SelArgs a{};
  a.imp = imp_out; a.row = N; a.pool_k = pool_k; a.chunk = chunk; a.pos0 = pos0; a.ppm = ppm;
  a.ids = ids; a.pos = pos; a.n_kept = n_kept; a.cs_ws = ws_scores(ws, B); a.tokens = tokens; a.out = out;
  a.n_glob = N;
  a.blk_cnt = ws_counters(ws);
  a.nreq = B;
  a.accp = accp; a.acc_pitch = pitch; a.n_ug = n_ug; a.Rv = Rv; a.imp_out = imp_out;
  long long nblk;
  size_t smem;
  if (!deferred_shape(a, N, Rv, n_ug, pool_k, chunk, &nblk, &smem)) return cudaErrorNotSupported;
  return launch_pdl<kPlain>(dim3(B, (unsigned)nblk), smem, st, a);
}

// Phases B-C only: the chunk scores were written into the workspace by the
// score kernel (sp_score_select).  One CTA per request, the scores staged in SMEM
// when they fit.
cudaError_t select_ready_launch(int B, long long N, int chunk, long long ppm, int pos0, int* ids, int* pos,
                                int* n_kept, void* ws, cudaStream_t st, const int* tokens, int* out) {
  cudaError_t e = configure<kPlain>();
  if (e != cudaSuccess) return e;
  SelArgs a{};
  a.imp = nullptr; a.row = N; a.pool_k = 1; a.chunk = chunk; a.pos0 = pos0; a.ppm = ppm;
  a.ids = ids; a.pos = pos; a.n_kept = n_kept; a.cs_ws = ws_scores(ws, B); a.tokens = tokens; a.out = out;
  a.n_glob = N;
  a.blk_cnt = ws_counters(ws);
  a.nreq = B;
  a.cs_ready = 1;
  a.mode = kModeAll;
  a.segcap = 0;
  a.cpb = 0;
  a.nblk = 1;
  const long long n_c = (N + chunk - 1) / chunk;
  const long long cs_floats = n_c <= kSmemChunks ? n_c : 0;
  a.sh_off = (int)((cs_floats + 3) / 4 * 4);
  return launch_pdl<kPlain>(dim3(B), (size_t)a.sh_off * sizeof(float) + sizeof(SelShared<ST>), st, a);
}

bool select_supported(int pool_k) { return pool_k <= kMaxPool; }

cudaError_t select_launch(const float* imp, int B, long long N, int pool_k, int chunk, int pos0, long long ppm,
                          int* ids, int* pos, int* n_kept, void* ws, cudaStream_t st, const int* tokens, int* out,
                          const int* seq_lens) {
  SelArgs a{};
  a.imp = imp; a.row = N; a.seq_lens = seq_lens; a.pool_k = pool_k; a.chunk = chunk; a.pos0 = pos0; a.ppm = ppm;
  a.ids = ids; a.pos = pos; a.n_kept = n_kept; a.cs_ws = ws_scores(ws, B); a.tokens = tokens; a.out = out;
  a.n_glob = N;
  a.blk_cnt = ws_counters(ws);
  return launch_select<kPlain>(a, B, N, (N + chunk - 1) / chunk, st);
}

long long seq_candidate_count(long long N, int world, int chunk, long long ppm) {
  const long long n_c = (N + chunk - 1) / chunk;
  const long long K_c = std::min(n_c, std::max(1LL, (ppm * n_c + 999999) / 1000000));
  return std::min(K_c, n_c / world);
}

size_t seq_select_ws_bytes(int B, long long N, int world, int chunk) {
  // kCand: the shard's chunk scores; kMerge: the prompt's (when above the SMEM limit); counters
  (void)world;
  return select_ws_bytes(B, N, chunk);
}

cudaError_t seq_edges_launch(const float* imp_local, int B, long long n_local, int pool_k, float* edges,
                             cudaStream_t st) {
  const int w = (pool_k - 1) / 2;
  if (w == 0) return cudaSuccess;
  k_seq_edges<<<B, 256, 0, st>>>(imp_local, n_local, w, edges);
  return cudaGetLastError();
}

cudaError_t seq_candidates_launch(const float* imp_local, const float* edges, int rank, int world, int B,
                                  long long N, int pool_k, int chunk, long long M, unsigned long long* cand, void* ws,
                                  cudaStream_t st) {
  const long long n_local = N / world;
  SelArgs a{};
  a.imp = imp_local; a.row = n_local; a.pool_k = pool_k; a.chunk = chunk;
  a.ids = nullptr; a.pos = nullptr; a.cs_ws = ws_scores(ws, B);
  a.i0 = (long long)rank * n_local; a.n_glob = N; a.edges = edges; a.rank = rank; a.world = world;
  a.k_sel = M; a.cand = cand;
  a.blk_cnt = ws_counters(ws);
  return launch_select<kCand>(a, B, n_local, n_local / chunk, st);
}

cudaError_t seq_merge_launch(const unsigned long long* cand_all, int world, int B, long long N, int pool_k, int chunk,
                             int pos0, long long ppm, long long M, const int* tokens, int* ids, int* pos, int* n_kept,
                             int* out, void* ws, cudaStream_t st) {
  SelArgs a{};
  a.row = N; a.pool_k = pool_k; a.chunk = chunk; a.pos0 = pos0; a.ppm = ppm;
  a.ids = ids; a.pos = pos; a.n_kept = n_kept; a.cs_ws = ws_scores(ws, B); a.tokens = tokens; a.out = out;
  a.n_glob = N; a.world = world; a.k_sel = M; a.cand_in = cand_all;
  a.blk_cnt = ws_counters(ws);
  return launch_select<kMerge>(a, B, N, (N + chunk - 1) / chunk, st);
}

}  // namespace sp
