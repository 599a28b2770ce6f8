/*
 * specprefill.h -- C ABI of the B200 (sm_100a) SpecPrefill hot path.
 *
 * SpecPrefill (arXiv 2502.02789) speculator-side token importance estimation
 * and selection: score -> aggregate -> pool -> chunked top-k -> gather.
 * Citations: P:n = line n of the paper's LaTeX with its section
 * label; Zk = reading k of the ambiguity register in DESIGN.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * Ownership   The caller owns every buffer.  Device pointers are plain
 *             cudaMalloc / PyTorch CUDA memory; the library never allocates
 *             or frees device memory on the hot path.  Scratch comes from a
 *             caller-provided workspace of at least *_workspace_bytes() bytes.
 *             A score workspace must be zero-filled before its first use with a
 *             given geometry (sp_geom) and may then be reused for that geometry
 *             indefinitely: the fused kernel's exchange counters are left at
 *             zero at the end of every successful call.  Reusing it for another
 *             geometry or another launch plan (sp_score_set_plan,
 *             sp_score_tune), or after SP_ETIMEOUT, requires zero-filling it
 *             again.
 * Streams     Every call is enqueued on `stream` (a cudaStream_t / CUstream;
 *             NULL = legacy default stream) and returns without synchronising.
 *             Outputs are valid in stream order.
 * Errors      Arguments are validated on the host before anything is
 *             launched; an invalid call returns a non-zero sp_status and
 *             touches nothing.  Device-side failures (non-finite softmax
 *             statistics, a stats exchange that never completes) set a
 *             device flag read by sp_check_device_error().  No C++ exception
 *             crosses this boundary.  There is no CPU fallback: a missing
 *             device or kernel is an error.
 * Determinism Same inputs, geometry and device give bit-identical outputs:
 *             every floating-point reduction has a fixed order.
 * Device      sm_100a (B200) only.
 */
#ifndef SPECPREFILL_H
#define SPECPREFILL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 1

typedef enum sp_status {
  SP_OK = 0,
  SP_EINVAL = 1,        /* invalid argument (shape, stride, alignment, keep rate, pool window, ...) */
  SP_EUNSUPPORTED = 2,  /* valid but no kernel for this geometry / device */
  SP_ECUDA = 3,         /* a CUDA runtime call failed */
  SP_ENONFINITE = 5,    /* device flag: a softmax statistic was not finite (Z15) */
  SP_EEMPTY = 6,        /* zero valid look-ahead rows */
  SP_EWORKSPACE = 7,    /* workspace too small or misaligned */
  SP_ETIMEOUT = 8       /* device flag: an in-kernel stats exchange timed out */
} sp_status;

/* A cudaStream_t / CUstream handle. */
typedef void* sp_stream;

/*
 * Geometry of one uniform batch (Alg.1 P:142-171 retrieve_qk: Q of the
 * look-ahead rows and K of the speculator KV cache C_s).
 *   B        requests in the batch (each is scored and selected independently)
 *   L        speculator layers
 *   H, Hkv   query / kv heads; H % Hkv == 0; query head h reads kv head h / (H/Hkv) (Z4)
 *   d        head dim; 16 <= d <= 256, d % 16 == 0
 *   R        captured query rows per request (look-ahead rows; Z1)
 *   R_valid  valid prefix of the rows (EOS check, Alg.1); 1 <= R_valid <= R
 *   N        prompt tokens per request (M in the paper's eq.)
 *   scale    softmax scale applied to q.k (Z3; 1/sqrt(d) for Llama)
 */
typedef struct sp_geom {
  int32_t B, L, H, Hkv, d;
  int32_t R, R_valid;
  int64_t N;
  float scale;
} sp_geom;

/*
 * Element strides (bf16 elements, not bytes) of the two inputs.  The head
 * dimension is always contiguous (stride 1).
 *   K[b][l][g][i][:]  at  K + b*k_b + l*k_l + g*k_g + i*k_i     (bf16)
 *   Q[b][l][r][h][:]  at  Q + b*q_b + l*q_l + r*q_r + h*q_h     (bf16)
 * Alignment: K, Q and every stride*2 bytes must be multiples of 16 bytes
 * (TMA tensor maps), strides must be non-negative, and a dimension of size > 1
 * may not have stride 0 (no broadcast views, e.g. K.expand(B, ...): SP_EINVAL).
 */
typedef struct sp_layout {
  int64_t k_b, k_l, k_g, k_i;
  int64_t q_b, q_l, q_r, q_h;
} sp_layout;

/*
 * Selection parameters (sec:chunk_select P:121-123, sec:position_ids P:125-133).
 *   keep_rate  ratio of chunks kept, (0, 1]; K_c = sp_kept_chunks(n_c, keep_rate)
 *   pool_k     odd 1-D average-pool window, 1 <= pool_k <= 4097, centred, shrinking at the edges (Z6)
 *   chunk      contiguous chunk size >= 1; the last chunk may be partial (Z8)
 *   pos0       position id of prompt token 0 (kept positions are ids + pos0)
 */
typedef struct sp_select_params {
  double keep_rate;
  int32_t pool_k;
  int32_t chunk;
  int32_t pos0;
} sp_select_params;

/* Score kernel choice. */
typedef enum sp_score_algo {
  SP_SCORE_AUTO = 0,   /* fused when supported, else SIMT */
  SP_SCORE_FUSED = 1,  /* tcgen05/TMA persistent kernel, logits TMEM-resident, one K read */
  SP_SCORE_SIMT = 2    /* two-pass FP32-FMA kernels (baseline; reads K twice) */
} sp_score_algo;

/* ------------------------------------------------------------------ utilities */
int sp_abi_version(void);
const char* sp_status_string(sp_status s);

/* K_c = clamp(ceil(keep_rate * n_chunks), 1, n_chunks), evaluated exactly on
 * keep_rate snapped to parts per million (Z9).  Returns -1 for an
 * invalid keep_rate or n_chunks < 1. */
int64_t sp_kept_chunks(int64_t n_chunks, double keep_rate);

/* Synchronises `stream`, then reads and clears the device error flag.
 * Returns SP_OK, SP_ENONFINITE, SP_ETIMEOUT or SP_ECUDA. */
sp_status sp_check_device_error(sp_stream stream);

/* Number of SMs the persistent kernels size their grid for (current device). */
int sp_device_sm_count(void);

/* ------------------------------------------------------------------ score
 * Token importance (O1-O4 in DESIGN.md):
 *   s[l,h,r,i]   = scale * <Q[b][l][r][h], K[b][l][h/G][i]>
 *   lse[l,h,r]   = log sum_i exp(s[l,h,r,i])   over the N prompt keys     (Z2)
 *   acc[r,i]     = max_{l,h} (s[l,h,r,i] - lse[l,h,r])                    (max over H and L)
 *   importance[b][i] = (1/R_valid) sum_{r<R_valid} exp(acc[r,i])          (mean over rows)
 * importance: device fp32 [B][N] (contiguous), written completely.
 * Q rows r >= R_valid are never read. */
size_t sp_score_workspace_bytes(const sp_geom* g, int algo);
sp_status sp_score(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay,
                   float* importance, void* ws, size_t ws_bytes, sp_stream stream);
sp_status sp_score_ex(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay,
                      float* importance, void* ws, size_t ws_bytes, int algo, sp_stream stream);

/* Launch plan of the fused kernel for g on the current device (for reports
 * and tests): out[0..9] = grid, jobs per request, token groups, unit groups,
 * tiles per job, units per job, TMEM unit slots, SMEM pipeline stages,
 * dynamic SMEM bytes, hierarchical exchange (0: every CTA of a unit polls the
 * unit's n_tg partial words; 1: the unit's last CTA merges them and the others
 * poll one word).  Returns SP_EUNSUPPORTED if the fused kernel cannot run g. */
sp_status sp_score_plan(const sp_geom* g, int64_t out[10]);

/* Measured plan choice.  sp_score_tune times the fused kernel's best model
 * candidates (token groups x unit groups; at most 6, within 1.3x of the model's
 * best) on this device with private workspaces (allocated and freed inside the
 * call: not for the hot path; synchronises `stream`) and registers the fastest
 * for g: every later sp_score / plan / workspace query of g uses it.  out[0..2]
 * = (token groups, unit groups, hierarchical); *ms_per_launch = its mean launch
 * time.  sp_score_set_plan registers a plan explicitly (n_tg = 0 clears; an
 * invalid plan is ignored at plan time).  After either call, re-query
 * sp_score_workspace_bytes(g) and use a freshly zero-filled workspace: the
 * partial-statistics layout depends on the plan. */
sp_status sp_score_tune(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, int64_t out[3],
                        float* ms_per_launch, sp_stream stream);
sp_status sp_score_set_plan(const sp_geom* g, int32_t n_tg, int32_t n_ug, int32_t hier);

/* Debug tracing of the fused kernel (not for production runs): while enabled,
 * every sp_score launch writes globaltimer stamps (ns) into device_buffer laid
 * out as [grid CTA][unit index within the CTA][8] uint64:
 *   0 producer starts the unit, 1 MMA starts it (TMEM slot free), 2 statistics
 *   start (logits in TMEM), 3 CTA partial published, 4 partials read (cleanup
 *   done), 5 lse2 combined from all partials, 6 aggregation done (TMEM slot
 *   released), 7 statistics compute done.
 * records = capacity in uint64; units beyond capacity are not traced.
 * device_buffer = NULL disables tracing. */
sp_status sp_trace_enable(uint64_t* device_buffer, int64_t records);

/* ------------------------------------------------------------------ score, sequence-sharded split
 * For a prompt split along tokens over P ranks.  Each
 * rank passes its own K shard (N = local tokens).  Statistics are in the log2
 * domain: x = s*log2(e);  m2 = max_i x;  l = sum_i 2^(x - m2).
 *   stats [B][L][H][R_valid][2] fp32 (m2, l) over the local tokens.
 * sp_stats_combine merges P gathered stats blocks [P][n_rows][2] in rank order
 * (deterministic) into lse2[n_rows] = m2 + log2(l), n_rows = B*L*H*R_valid.
 * sp_score_finish computes importance over the local tokens given the global
 * lse2 (same formula as sp_score). */
size_t sp_score_split_workspace_bytes(const sp_geom* g);
sp_status sp_score_stats(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay,
                         float* stats, void* ws, size_t ws_bytes, sp_stream stream);
sp_status sp_stats_combine(const float* parts, int32_t P, int64_t n_rows, float* lse2, sp_stream stream);
sp_status sp_score_finish(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay,
                          const float* lse2, float* importance, void* ws, size_t ws_bytes, sp_stream stream);

/* ------------------------------------------------------------------ score, head-sharded partition
 * the (l, h)-max of O3 is
 * order-free, so the query heads (with their kv heads: H and Hkv divided by the
 * same P, G unchanged) can be split over P ranks.  Each rank passes its own
 * Q/K heads; every lse is complete on its rank (all N tokens are local), so
 * the only exchange is an elementwise MAX of
 *   acc2 [B][R_valid][N] fp32 = max_{local l,h} (x - lse2)   (log2 domain, x = s*log2 e)
 * followed by sp_acc_importance: importance[b][i] = (1/R_valid) sum_r 2^acc2[b][r][i]
 * (the fused kernel's own epilogue arithmetic).  sp_score_acc runs the fused
 * kernel only (SP_EUNSUPPORTED otherwise); its workspace is
 * sp_score_workspace_bytes(g, SP_SCORE_FUSED).  acc2 is written for every
 * valid (b, r, i); the caller owns it. */
sp_status sp_score_acc(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, float* acc2,
                       void* ws, size_t ws_bytes, sp_stream stream);
sp_status sp_acc_importance(const float* acc2, int32_t B, int32_t R_valid, int64_t N, float* importance,
                            sp_stream stream);

/* ------------------------------------------------------------------ score, sequence-sharded single pass
 * The prompt split along tokens over `world` ranks (<= 8), one launch per rank,
 * K read once: the fused kernel's per-unit softmax-statistics exchange runs
 * over peer memory, hierarchically.  Each CTA publishes its 64-bit (max2, sum)
 * partial words into its own rank's workspace; the last CTA of a unit on rank
 * r to publish merges the rank's n_tg partials in token-group order and stores
 * the rank's word into row r of EVERY rank's rank-word buffer (NVLink stores,
 * st.relaxed.sys); every CTA polls the unit's `world` rank words from its own
 * buffer and merges them in rank order, so every rank computes the same lse2
 * bit for bit.  The importance of the rank's own tokens is written to
 * importance [B][N_local].
 * peer_buffers: host array of `world` device pointers (256-B aligned), entry r =
 * rank r's rank-word buffer of sp_score_peer_buffer_bytes(g, world, sm_budget)
 * bytes, mapped into this process (e.g. torch symmetric memory), zero-filled
 * once before first use (the kernel keeps it so).  All ranks pass the same
 * geometry (equal shards), world and sm_budget, and their launches of one call
 * must be co-resident (they wait for each other inside the kernel; a missing
 * rank ends in a device timeout, SP_ETIMEOUT from sp_check_device_error).
 * Consecutive calls must be separated by a cross-rank barrier (the sequence-
 * sharded selection's edge all-gather that follows is one).  sm_budget > 0 caps
 * the CTAs per launch (0 = every SM), so several "ranks" can share one GPU (the
 * virtual-rank tests).  ws: a private workspace of
 * sp_score_peer_workspace_bytes(g, world, sm_budget) bytes, zero-filled once and
 * kept with the peer buffers (its launch epoch selects the buffers' half).
 * sp_score_peer_plan reports the plan (as sp_score_plan) for world ranks under
 * sm_budget. */
size_t sp_score_peer_buffer_bytes(const sp_geom* g, int32_t world, int32_t sm_budget);
size_t sp_score_peer_workspace_bytes(const sp_geom* g, int32_t world, int32_t sm_budget);
sp_status sp_score_peer_plan(const sp_geom* g, int32_t world, int32_t sm_budget, int64_t out[10]);
sp_status sp_score_peer(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, int32_t rank,
                        int32_t world, void* const* peer_buffers, int32_t sm_budget, float* importance, void* ws,
                        size_t ws_bytes, sp_stream stream);

/* ------------------------------------------------------------------ score, FP8 (e4m3) inputs
 * SURVEY 8(f) row f4 (an FP8 KV cache halves the K bytes, the path's cost).
 * Q8, K8 hold OCP FP8 E4M3 codes (1 byte: sign, 4 exponent bits with bias 7,
 * 3 mantissa bits; S.1111.111 is NaN, no infinities) with per-tensor
 * dequantisation scales: Q = q_scale * e4m3(Q8), K = k_scale * e4m3(K8) (the
 * usual FP8 attention formulation).  The scores are those of sp_score on these
 * dequantised values, s = scale * <Q, K>, computed as
 * (scale*q_scale*k_scale) * <e4m3(Q8), e4m3(K8)> with e4m3 x e4m3 products
 * (exact in fp32) on the tensor cores (tcgen05.mma kind::f8f6f4), fp32
 * accumulation; everything after the logits is sp_score's fused kernel.
 * Layout: sp_layout strides in elements = bytes; rows 16-byte aligned;
 * d % 32 == 0 (else SP_EUNSUPPORTED).  q_scale, k_scale finite and > 0.
 * Workspace: sp_score_e4m3_workspace_bytes(g) bytes, same rules as sp_score. */
size_t sp_score_e4m3_workspace_bytes(const sp_geom* g);
sp_status sp_score_e4m3_plan(const sp_geom* g, int64_t out[10]);
sp_status sp_score_e4m3(const void* Q8, const void* K8, float q_scale, float k_scale, const sp_geom* g,
                        const sp_layout* lay, float* importance, void* ws, size_t ws_bytes, sp_stream stream);
/* sp_score_tune for the e4m3 path (its plans are registered separately from bf16's). */
sp_status sp_score_e4m3_tune(const void* Q8, const void* K8, float q_scale, float k_scale, const sp_geom* g,
                             const sp_layout* lay, int64_t out[3], float* ms_per_launch, sp_stream stream);

/* ------------------------------------------------------------------ score, look-ahead-key denominator
 * SURVEY 8(f) row f4, reading Z2': each look-ahead
 * row's softmax also covers the look-ahead tokens' own keys -- "softmax over
 * ALL keys visible to that row (context plus any earlier decoded tokens) ...
 * sliced to the first M context entries WITHOUT renormalization".  Row r sees
 * the N prompt keys and K_la[b][l][g][j] for j <= r - la_shift (causal):
 * la_shift = 0 when row r is the r-th look-ahead token (its own key is
 * K_la[.., r]); 1 when row 0 is the last prompt token (whose key is in K) and
 * row r >= 1 the r-th decoded token (key K_la[.., r - 1]).
 *   s_la[j] = scale * <Q[b][l][r][h], K_la[b][l][h/G][j]>
 *   lse'    = log( sum_i exp(s[i]) + sum_{j <= r - la_shift} exp(s_la[j]) )
 *   acc[r,i] = max_{l,h} (s[l,h,r,i] - lse'),  importance = mean_r exp(acc)
 * K_la: bf16, element strides s_b, s_l, s_g, s_j (d contiguous), at least
 * R_valid - la_shift rows per (b, l, g).  Fused kernel only; workspace
 * sp_score_lookahead_workspace_bytes(g) bytes (zero-filled once, as sp_score's). */
typedef struct sp_lookahead_k {
  const void* K_la;
  int64_t s_b, s_l, s_g, s_j;
  int32_t la_shift;
} sp_lookahead_k;

size_t sp_score_lookahead_workspace_bytes(const sp_geom* g);
sp_status sp_score_lookahead(const void* Q, const void* K, const sp_lookahead_k* la, const sp_geom* g,
                             const sp_layout* lay, float* importance, void* ws, size_t ws_bytes, sp_stream stream);

/* ------------------------------------------------------------------ score, paged K cache / ragged batch
 * the speculator's K cache in the serving layout -- fixed-size
 * blocks addressed through a block table (the "slot mapping" of the paper's vLLM
 * integration; Alg.1) -- and requests of different prompt lengths.
 * Per layer l the cache holds num_blocks blocks of block_size tokens:
 *   K[l][blk][j][g][:]  at  cache + l*s_l + blk*s_blk + j*s_tok + g*s_g   (bf16, d contiguous)
 * (vLLM's per-layer [num_blocks][block_size][Hkv][d] key cache with a uniform
 * layer stride, e.g. one allocation for all layers).  Token i of request b is
 * row i % block_size of physical block block_table[b][i / block_size].
 *   block_size   a power of two >= 8 (8 ... 64 divide a 128-token tile; >= 128 hold whole tiles)
 *   block_table  device int32 [B][max_blocks], max_blocks >= ceil(N / block_size);
 *                entries past a request's last block are never read
 *   seq_lens     device int32 [B]: request b's prompt length n_b (clamped to [1, N]),
 *                or NULL: every request has N tokens.  g->N is the longest length.
 * Scores are sp_score's over each request's own n_b tokens
 * (softmax over its prompt keys only).  importance [B][N]: entries i < n_b are
 * written, the rest of each row is left untouched.  Q and sp_layout's q_*
 * strides as for sp_score (k_* are ignored).  Fused kernel only
 * (SP_EUNSUPPORTED otherwise); workspace sp_score_paged_workspace_bytes(g),
 * same rules as sp_score.  Alignment: cache and every stride*2 bytes multiples
 * of 16 bytes. */
typedef struct sp_paged_k {
  const void* cache;
  int64_t s_l, s_blk, s_tok, s_g;
  int32_t num_blocks, block_size;
  const int32_t* block_table;
  int32_t max_blocks;
  const int32_t* seq_lens;
} sp_paged_k;

size_t sp_score_paged_workspace_bytes(const sp_geom* g);
sp_status sp_score_paged(const void* Q, const sp_paged_k* K, const sp_geom* g, const sp_layout* lay,
                         float* importance, void* ws, size_t ws_bytes, sp_stream stream);

/* Rows f3 x f4: a paged FP8 cache (vLLM's fp8 KV cache) -- Q8 and the cache hold
 * e4m3 codes with per-tensor scales as in sp_score_e4m3; strides in elements =
 * bytes (multiples of 16), d % 32 == 0.  Workspace sp_score_e4m3_workspace_bytes(g). */
sp_status sp_score_paged_e4m3(const void* Q8, const sp_paged_k* K, float q_scale, float k_scale, const sp_geom* g,
                              const sp_layout* lay, float* importance, void* ws, size_t ws_bytes, sp_stream stream);

/* ------------------------------------------------------------------ select
 * Pool, chunk means, top-K_c chunks, positions (O5-O9, Alg.1):
 *   pooled[i] = mean(importance[j] : |j-i| <= (pool_k-1)/2, 0 <= j < N)      (Z6)
 *   cs[c]     = mean(pooled[c*chunk .. min(N,(c+1)*chunk)-1])                 (Z8)
 *   keep the K_c chunks first in (cs desc, c asc) order                       (Z10)
 *   ids  = ascending union of the kept chunks' token indices                  (Z11)
 *   pos  = ids + pos0;  the first decode position is N + pos0
 * importance: device fp32 [B][N].  ids, pos: device int32 [B][N] (capacity N per
 * request; entries >= n_kept[b] are left untouched).  n_kept: device int32 [B].
 * Workspace: sp_select_workspace_bytes bytes, zero-filled once before first use
 * (it holds per-request completion counters that the kernel leaves at zero),
 * not shared by concurrent calls.  One launch, programmatic-dependent on the
 * preceding kernel of the stream (it waits for that kernel's results inside). */
size_t sp_select_workspace_bytes(int32_t B, int64_t N, const sp_select_params* p);
sp_status sp_select(const float* importance, int32_t B, int64_t N, const sp_select_params* p,
                    int32_t* ids, int32_t* pos, int32_t* n_kept, void* ws, size_t ws_bytes,
                    sp_stream stream);

/* sp_select + sp_gather in one launch: additionally out_tokens[b][j] =
 * tokens[b][ids[b][j]] for j < n_kept[b] (bit-exact).  tokens / out_tokens:
 * device int32 [B][N]; both NULL is the same as sp_select. */
sp_status sp_select_gather(const float* importance, const int32_t* tokens, int32_t B, int64_t N,
                           const sp_select_params* p, int32_t* ids, int32_t* pos, int32_t* n_kept,
                           int32_t* out_tokens, void* ws, size_t ws_bytes, sp_stream stream);

/* Ragged batch (row f3): sp_select_gather over per-request prompt lengths.
 * seq_lens: device int32 [B], n_b clamped to [1, N]; request b's selection is
 * the one above over importance[b][0 .. n_b) with n_c = ceil(n_b / chunk) and
 * K_c = sp_kept_chunks(n_c, keep_rate) (evaluated on the device with the same
 * integer rule).  Rows of every [B][N] array keep their stride N.  tokens /
 * out_tokens may both be NULL. */
sp_status sp_select_ragged(const float* importance, const int32_t* seq_lens, const int32_t* tokens, int32_t B,
                           int64_t N, const sp_select_params* p, int32_t* ids, int32_t* pos, int32_t* n_kept,
                           int32_t* out_tokens, void* ws, size_t ws_bytes, sp_stream stream);

/* ------------------------------------------------------------------ score + select in one call
 * sp_score followed by sp_select_gather (O1-O11, Alg.1) with the same
 * outputs, bit for bit, in one call: the score kernel, then the selection
 * launched as its programmatic dependent.  When the fused plan splits a token
 * group over >= 2 unit groups, the score kernel leaves its cross-unit-group
 * max (the "maximum over H and L" of sec:attn_agg) as partial maps in
 * the workspace and the selection launch finalizes the importance from them
 * (the same instruction, the same order: `importance` is still written, bit-
 * identical to sp_score's) before pooling and ranking -- the epilogue's chain
 * of cross-CTA round trips leaves the score kernel's tail.
 * Workspace: sp_score_select_workspace_bytes(g, p) bytes, 256-byte aligned,
 * zero-filled once and reused only for this geometry and selection.  tokens /
 * out_tokens may both be NULL (no gather). */
size_t sp_score_select_workspace_bytes(const sp_geom* g, const sp_select_params* p);
sp_status sp_score_select(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay,
                          const sp_select_params* p, const int32_t* tokens, float* importance, int32_t* ids,
                          int32_t* pos, int32_t* n_kept, int32_t* out_tokens, void* ws, size_t ws_bytes,
                          sp_stream stream);

/* The score kernel with the selection's pooling and chunk means in its
 * epilogue (each token group's chunks once its importance and its neighbours'
 * are written; the measured alternative to the deferred finalize, DESIGN.md
 * 5.3): the importance (as sp_score) plus the chunk scores cs[b][c] = mean over chunk c of the pooled
 * importance (O5-O6: centred window of pool_k with shrinking edges, Z6; the
 * partial last chunk over its true size, Z8), c < ceil(N / chunk), the same bits
 * as the selection computes -- for callers that rank the chunks themselves.
 * cs: device float [B][ceil(N / chunk)].  pool_k odd, 1..4097; chunk 1..16384.
 * Workspace: sp_score_workspace_bytes(g).  SP_EUNSUPPORTED when the geometry's
 * plan cannot stage a token group's window in the epilogue (then sp_score +
 * sp_select). */
sp_status sp_score_chunks(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, int32_t pool_k,
                          int32_t chunk, float* importance, float* cs, void* ws, size_t ws_bytes, sp_stream stream);

/* ------------------------------------------------------------------ sequence-sharded select
 * Row e: one request's prompt split along tokens over
 * P ranks (the paper's TP=8 placement), rank p holding the
 * importance of tokens [p*N/P, (p+1)*N/P).  The selection of O5-O9 (Alg.1 P:163,
 * chunk_select_from_smoothed_attention) is computed without gathering the
 * importance vector:
 *   1. sp_seq_edges: this rank's first w and last w importance values
 *      (w = (pool_k-1)/2), edges [B][2w];
 *   2. the caller all-gathers them -> edges_all [P][B][2w] (rank order);
 *   3. sp_seq_candidates: pool (windows reach into the neighbours' edges), chunk
 *      means and the local top M = min(K_c, n_c/P) chunks in (cs desc, c asc)
 *      order, written in chunk order as 64-bit keys (float bits of cs << 32 |
 *      ~global chunk index): compared as unsigned integers they follow the
 *      same total order; cand [B][M];
 *   4. the caller all-gathers them -> cand_all [P][B][M];
 *   5. sp_seq_merge: the global top-K_c of the P*M candidates (identical on
 *      every rank) -> ids / pos / n_kept for the whole prompt, as sp_select
 *      writes them, and the gathered tokens when tokens (replicated [B][N]) is
 *      given.  The global top-K_c is contained in the union of the local top-M
 *      lists because every rank ranks by the same total order.
 * Chunk scores are computed in the same order as sp_select's, so for the same
 * importance values the result is bit-identical to sp_select_gather on the
 * concatenated vector.  Requires N % P == 0, (N/P) % chunk == 0 and
 * w <= N/P (SP_EINVAL otherwise).  All device buffers are caller-owned. */
int64_t sp_seq_candidate_count(int64_t N, int32_t world, const sp_select_params* p);   /* M, or -1 if invalid */
size_t sp_seq_select_workspace_bytes(int32_t B, int64_t N, int32_t world, const sp_select_params* p);
sp_status sp_seq_edges(const float* imp_local, int32_t B, int64_t N, int32_t world, const sp_select_params* p,
                       float* edges, sp_stream stream);
sp_status sp_seq_candidates(const float* imp_local, const float* edges_all, int32_t rank, int32_t world, int32_t B,
                            int64_t N, const sp_select_params* p, uint64_t* cand, void* ws, size_t ws_bytes,
                            sp_stream stream);
sp_status sp_seq_merge(const uint64_t* cand_all, int32_t world, int32_t B, int64_t N, const sp_select_params* p,
                       const int32_t* tokens, int32_t* ids, int32_t* pos, int32_t* n_kept, int32_t* out_tokens,
                       void* ws, size_t ws_bytes, sp_stream stream);

/* ------------------------------------------------------------------ gather
 * out[b][j] = tokens[b][ids[b][j]] for j < n_kept[b] (merge_requests input,
 * Alg.1).  tokens, ids, out: device int32 [B][N]; n_kept device int32 [B].
 * Bit-exact. */
sp_status sp_gather(const int32_t* tokens, const int32_t* ids, const int32_t* n_kept, int32_t B,
                    int64_t N, int32_t* out, sp_stream stream);

/* ------------------------------------------------------------------ end to end from host buffers
 * The whole path with host inputs/outputs: copies Q, K and tokens host->device,
 * runs sp_score -> sp_select_gather, copies ids, pos, n_kept and the
 * gathered tokens device->host, all enqueued on `stream` (host buffers should
 * be pinned for the copies to be asynchronous).  Host Q/K use the same element
 * strides `lay` as the device copies; host outputs are [B][N] / [B]. */
typedef struct sp_host_io {
  const void* Q;
  const void* K;
  const int32_t* tokens;
  int32_t* ids;
  int32_t* pos;
  int32_t* n_kept;
  int32_t* out_tokens;
  size_t q_bytes;   /* bytes of Q / K to copy (span of the strided layout) */
  size_t k_bytes;
} sp_host_io;

typedef struct sp_device_bufs {
  void* Q;
  void* K;
  int32_t* tokens;
  float* importance;
  int32_t* ids;
  int32_t* pos;
  int32_t* n_kept;
  int32_t* out_tokens;
  void* ws;
  size_t ws_bytes;
} sp_device_bufs;

size_t sp_run_workspace_bytes(const sp_geom* g, const sp_select_params* p);
sp_status sp_run_host(const sp_host_io* host, const sp_device_bufs* dev, const sp_geom* g,
                      const sp_layout* lay, const sp_select_params* p, sp_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECPREFILL_H */
