// Internal declarations shared by the translation units of libspecprefill.so.
// Not part of the ABI (include/specprefill.h is).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/specprefill.h"

namespace sp {

// log2(e): the kernels work in the log2 domain, x = s * log2(e), so that
// exp(s - lse) == exp2(x - lse2) with one ex2 per probability.
constexpr float kLog2e = 1.4426950408889634f;

// Device error codes written into the device flag (first error wins).
enum DevErr : int { kDevOk = 0, kDevNonFinite = 1, kDevTimeout = 2 };

// Pointer to this device's error flag (int), resolved once per device.
int* device_error_flag();

struct Geom {
  int B, L, H, Hkv, d, R, Rv, G;
  long long N;
  float scale;
  int esz = 2;          // input element bytes: 2 = bf16, 1 = e4m3 (row f4; scale then folds q_scale*k_scale)
};

struct Layout {
  long long k_b, k_l, k_g, k_i;
  long long q_b, q_l, q_r, q_h;
};

inline Geom to_geom(const sp_geom& g) {
  Geom o;
  o.B = g.B; o.L = g.L; o.H = g.H; o.Hkv = g.Hkv; o.d = g.d; o.R = g.R; o.Rv = g.R_valid;
  o.G = g.H / g.Hkv; o.N = g.N; o.scale = g.scale;
  return o;
}
inline Layout to_layout(const sp_layout& l) {
  Layout o;
  o.k_b = l.k_b; o.k_l = l.k_l; o.k_g = l.k_g; o.k_i = l.k_i;
  o.q_b = l.q_b; o.q_l = l.q_l; o.q_r = l.q_r; o.q_h = l.q_h;
  return o;
}

// Row f3: a paged K cache (element strides; d contiguous) + block table + lengths.
struct PagedK {
  const void* cache;
  long long s_l, s_blk, s_tok, s_g;
  int num_blocks, bs;
  const int* btab;
  int max_blocks;
  const int* seq_lens;
};

// Z2' (row f4): the look-ahead tokens' keys K_la[b][l][g][j][:] (element strides).
struct LookaheadK {
  const void* K;
  long long s_b, s_l, s_g, s_j;
  int shift;
};

// Selection phase A run by the score kernel's epilogue (sp_score_select): the
// chunk scores go to cs ([B][ceil(N / chunk)], the selection workspace's).
struct ChunkOut {
  float* cs;
  int pool_k, chunk;
};

// Round up to a multiple of 256 bytes (workspace carving).
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------------- SIMT score (score_simt.cu)
size_t simt_score_ws_bytes(const Geom& g);
size_t simt_split_ws_bytes(const Geom& g);
// full single-device score: stats -> combine -> finish -> importance
cudaError_t simt_score(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                       float* importance, void* ws, cudaStream_t st);
// split API pieces
cudaError_t simt_score_stats(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                             float* stats, void* ws, cudaStream_t st);
cudaError_t stats_combine(const float* parts, int P, long long n_rows, float* lse2, cudaStream_t st);
cudaError_t simt_score_finish(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                              const float* lse2, float* importance, void* ws, cudaStream_t st);

// ---------------------------------------------------------------- fused tcgen05 score (score_fused.cu)
bool fused_supported(const Geom& g, const Layout& lay, const void* Q, const void* K);
// plan summary: grid, jobs/request, n_tg, n_ug, tiles/job, units/job, TMEM slots, stages, SMEM bytes, hier
constexpr int kPlanInfo = 10;
size_t fused_score_ws_bytes(const Geom& g);
bool fused_plan_info(const Geom& g, long long out[kPlanInfo]);
void fused_set_trace(unsigned long long* buf, long long records);
cudaError_t fused_score(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                        float* importance, void* ws, size_t ws_bytes, cudaStream_t st);
// the importance plus the selection's chunk scores (cudaErrorNotSupported: this
// geometry / plan cannot stage them; the caller runs the plain score + selection)
cudaError_t fused_score_chunks(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                               float* importance, const ChunkOut& co, void* ws, size_t ws_bytes, cudaStream_t st);
// the score kernel without its cross-unit-group epilogue: *accp ([B][n_ug][Rv][*pitch]
// in ws) holds the unit groups' partial maps for select_deferred_launch
// (cudaErrorNotSupported: the plan has one unit group)
cudaError_t fused_score_deferred(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                                 void* ws, size_t ws_bytes, cudaStream_t st, const float** accp, int* n_ug,
                                 long long* pitch);
cudaError_t fused_score_stats(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                              float* stats, void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t fused_score_finish(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                               const float* lse2, float* importance, void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t fused_score_acc(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                            float* acc2, void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t fused_score_paged(const __nv_bfloat16* Q, const PagedK& K, const Geom& g, const Layout& lay,
                              float* importance, void* ws, size_t ws_bytes, cudaStream_t st);
size_t fused_la_ws_bytes(const Geom& g);
cudaError_t fused_score_la(const __nv_bfloat16* Q, const __nv_bfloat16* K, const LookaheadK& la, const Geom& g,
                           const Layout& lay, float* importance, void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t fused_tune(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                       cudaStream_t st, int* tg_out, int* ug_out, int* hier_out, float* ms_out);
bool fused_set_plan(const Geom& g, int n_tg, int n_ug, int hier);
cudaError_t acc_importance(const float* acc2, int B, int Rv, long long N, float* importance, cudaStream_t st);
size_t fused_peer_buffer_bytes(const Geom& g, int world, int sm_budget);
size_t fused_peer_ws_bytes(const Geom& g, int world, int sm_budget);
bool fused_peer_plan_info(const Geom& g, int world, int sm_budget, long long out[kPlanInfo]);
cudaError_t fused_score_peer(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                             int rank, int world, void* const* bufs, int sm_budget, float* importance, void* ws,
                             size_t ws_bytes, cudaStream_t st);

// ---------------------------------------------------------------- select / gather (select.cu, gather.cu)
size_t select_ws_bytes(int B, long long N, int chunk);
bool select_supported(int pool_k);
// ppm: keep rate in parts per million (K_c per request, Z9); seq_lens: optional
// device [B] per-request prompt lengths (row f3), rows of the arrays stay N long
cudaError_t select_launch(const float* imp, int B, long long N, int pool_k, int chunk, int pos0,
                          long long ppm, int* ids, int* pos, int* n_kept, void* ws, cudaStream_t st,
                          const int* tokens = nullptr, int* out = nullptr, const int* seq_lens = nullptr);
// phases B-C over chunk scores already in the workspace (sp_score_select)
cudaError_t select_ready_launch(int B, long long N, int chunk, long long ppm, int pos0, int* ids, int* pos,
                                int* n_kept, void* ws, cudaStream_t st, const int* tokens, int* out);
float* select_ws_scores(void* ws, int B);
// the selection finalizing a deferred score launch's importance (written to imp_out)
bool select_deferred_supported(long long N, int Rv, int n_ug, int pool_k, int chunk);
cudaError_t select_deferred_launch(const float* accp, long long pitch, int n_ug, int Rv, float* imp_out, int B, long long N,
                                   int pool_k, int chunk, int pos0, long long ppm, int* ids, int* pos, int* n_kept,
                                   void* ws, cudaStream_t st, const int* tokens, int* out);
// sequence-sharded selection (row e)
long long seq_candidate_count(long long N, int world, int chunk, long long ppm);
size_t seq_select_ws_bytes(int B, long long N, int world, int chunk);
cudaError_t seq_edges_launch(const float* imp_local, int B, long long n_local, int pool_k, float* edges,
                             cudaStream_t st);
cudaError_t seq_candidates_launch(const float* imp_local, const float* edges, int rank, int world, int B,
                                  long long N, int pool_k, int chunk, long long M, unsigned long long* cand, void* ws,
                                  cudaStream_t st);
cudaError_t seq_merge_launch(const unsigned long long* cand_all, int world, int B, long long N, int pool_k, int chunk,
                             int pos0, long long ppm, long long M, const int* tokens, int* ids, int* pos, int* n_kept,
                             int* out, void* ws, cudaStream_t st);
cudaError_t gather_launch(const int* tokens, const int* ids, const int* n_kept, int B, long long N, int* out,
                          cudaStream_t st);

}  // namespace sp
