// C ABI of libspecprefill.so (declared in include/specprefill.h).
//
// Host-side argument validation, workspace carving and kernel dispatch.  No
// exception crosses this boundary; every entry point returns an sp_status.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "sp_internal.h"

namespace sp {

__device__ int g_sp_err;      // device error flag (DevErr), one per device

int* device_error_flag() {
  static int* ptrs[64] = {nullptr};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (ptrs[dev] == nullptr) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_sp_err) != cudaSuccess) return nullptr;
    ptrs[dev] = reinterpret_cast<int*>(p);
  }
  return ptrs[dev];
}

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// sm_100 device present and current?
sp_status check_device() {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return SP_ECUDA; }
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
    cudaGetLastError();
    return SP_ECUDA;
  }
  if (major != 10 || minor != 0) return SP_EUNSUPPORTED;   // sm_100a only
  return SP_OK;
}

sp_status check_geom(const sp_geom* g) {
  if (g == nullptr) return SP_EINVAL;
  if (g->B < 1 || g->L < 1 || g->H < 1 || g->Hkv < 1 || g->R < 1 || g->N < 1) return SP_EINVAL;
  if (g->H % g->Hkv != 0) return SP_EINVAL;
  if (g->d < 16 || g->d > 256 || g->d % 16 != 0) return SP_EINVAL;
  if (g->R_valid < 0 || g->R_valid > g->R) return SP_EINVAL;
  if (g->R_valid == 0) return SP_EEMPTY;
  if (!(std::isfinite(g->scale) && g->scale > 0.f)) return SP_EINVAL;
  if (g->N >= (1LL << 31)) return SP_EINVAL;
  return SP_OK;
}

// esz: element bytes of Q and K (2 = bf16, 1 = e4m3)
sp_status check_layout(const sp_geom* g, const sp_layout* l, const void* Q, const void* K, int esz = 2) {
  if (l == nullptr || Q == nullptr || K == nullptr) return SP_EINVAL;
  const long long ks[4] = {l->k_b, l->k_l, l->k_g, l->k_i};
  const long long kn[4] = {g->B, g->L, g->Hkv, g->N};
  const long long qs[4] = {l->q_b, l->q_l, l->q_r, l->q_h};
  const long long qn[4] = {g->B, g->L, g->R, g->H};
  for (int i = 0; i < 4; ++i) {
    if (ks[i] < 0 || qs[i] < 0) return SP_EINVAL;
    if (kn[i] > 1 && (ks[i] * esz) % 16 != 0) return SP_EINVAL;   // TMA: strides multiple of 16 B
    if (qn[i] > 1 && (qs[i] * esz) % 16 != 0) return SP_EINVAL;
    if ((kn[i] > 1 && ks[i] == 0) || (qn[i] > 1 && qs[i] == 0)) return SP_EINVAL;   // no broadcast (stride-0) dims
  }
  if (l->k_i < g->d && g->N > 1) return SP_EINVAL;               // rows of one head may not overlap
  if (!aligned16(Q) || !aligned16(K)) return SP_EINVAL;
  return SP_OK;
}

sp_status check_select(int32_t B, int64_t N, const sp_select_params* p) {
  if (p == nullptr || B < 1 || N < 1 || N >= (1LL << 31)) return SP_EINVAL;
  if (!(p->keep_rate > 0.0 && p->keep_rate <= 1.0)) return SP_EINVAL;
  if (p->pool_k < 1 || p->pool_k % 2 == 0) return SP_EINVAL;
  if (p->chunk < 1) return SP_EINVAL;
  if (!select_supported(p->pool_k)) return SP_EUNSUPPORTED;
  if (p->pos0 < 0 || (long long)p->pos0 + N >= (1LL << 31)) return SP_EINVAL;
  return SP_OK;
}

// keep rate snapped to parts per million (Z9); the kernels evaluate
// K_c = clamp(ceil(ppm * n_c / 1e6), 1, n_c) in integers, as sp_kept_chunks does
long long keep_ppm(double keep_rate) { return (long long)std::floor(keep_rate * 1000000.0 + 0.5); }

sp_status from_cuda(cudaError_t e) {
  if (e == cudaSuccess) return SP_OK;
  cudaGetLastError();
  return SP_ECUDA;
}

int resolve_algo(const Geom& g, int algo) {
  if (algo == SP_SCORE_AUTO) return fused_supported(g, Layout{}, nullptr, nullptr) ? SP_SCORE_FUSED : SP_SCORE_SIMT;
  return algo;
}

size_t score_ws(const Geom& g, int algo) {
  algo = resolve_algo(g, algo);
  return algo == SP_SCORE_FUSED ? fused_score_ws_bytes(g) : simt_score_ws_bytes(g);
}

}  // namespace
}  // namespace sp

using namespace sp;

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }

const char* sp_status_string(sp_status s) {
  switch (s) {
    case SP_OK: return "SP_OK";
    case SP_EINVAL: return "SP_EINVAL: invalid argument";
    case SP_EUNSUPPORTED: return "SP_EUNSUPPORTED: no kernel for this geometry/device (sm_100a required)";
    case SP_ECUDA: return "SP_ECUDA: CUDA runtime error";
    case SP_ENONFINITE: return "SP_ENONFINITE: non-finite softmax statistic";
    case SP_EEMPTY: return "SP_EEMPTY: zero valid look-ahead rows";
    case SP_EWORKSPACE: return "SP_EWORKSPACE: workspace too small or misaligned";
    case SP_ETIMEOUT: return "SP_ETIMEOUT: in-kernel statistics exchange timed out";
  }
  return "SP_?: unknown status";
}

int64_t sp_kept_chunks(int64_t n_chunks, double keep_rate) {
  if (n_chunks < 1 || !(keep_rate > 0.0 && keep_rate <= 1.0)) return -1;
  const long long ppm = keep_ppm(keep_rate);
  long long k = (ppm * n_chunks + 999999) / 1000000;
  if (k < 1) k = 1;
  if (k > n_chunks) k = n_chunks;
  return k;
}

int sp_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}

sp_status sp_check_device_error(sp_stream stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cudaStreamSynchronize(st) != cudaSuccess) { cudaGetLastError(); return SP_ECUDA; }
  int v = 0, zero = 0;
  if (cudaMemcpyFromSymbol(&v, g_sp_err, sizeof(int)) != cudaSuccess) { cudaGetLastError(); return SP_ECUDA; }
  if (v != 0 && cudaMemcpyToSymbol(g_sp_err, &zero, sizeof(int)) != cudaSuccess) { cudaGetLastError(); return SP_ECUDA; }
  if (v == kDevNonFinite) return SP_ENONFINITE;
  if (v == kDevTimeout) return SP_ETIMEOUT;
  return SP_OK;
}

size_t sp_score_workspace_bytes(const sp_geom* g, int algo) {
  if (check_geom(g) != SP_OK) return 0;
  return score_ws(to_geom(*g), algo);
}

sp_status sp_score_ex(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, float* importance,
                      void* ws, size_t ws_bytes, int algo, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if (importance == nullptr) return SP_EINVAL;
  if (algo != SP_SCORE_AUTO && algo != SP_SCORE_FUSED && algo != SP_SCORE_SIMT) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  Geom G = to_geom(*g);
  Layout Lay = to_layout(*lay);
  algo = resolve_algo(G, algo);
  if (algo == SP_SCORE_FUSED && !fused_supported(G, Lay, Q, K)) return SP_EUNSUPPORTED;
  const size_t need = score_ws(G, algo);
  if (ws == nullptr || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return SP_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(Q);
  const __nv_bfloat16* k = reinterpret_cast<const __nv_bfloat16*>(K);
  if (algo == SP_SCORE_FUSED) return from_cuda(fused_score(q, k, G, Lay, importance, ws, ws_bytes, st));
  return from_cuda(simt_score(q, k, G, Lay, importance, ws, st));
}

sp_status sp_score(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, float* importance, void* ws,
                   size_t ws_bytes, sp_stream stream) {
  return sp_score_ex(Q, K, g, lay, importance, ws, ws_bytes, SP_SCORE_AUTO, stream);
}

sp_status sp_score_acc(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, float* acc2, void* ws,
                       size_t ws_bytes, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if (acc2 == nullptr) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  const Geom G = to_geom(*g);
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q, K)) return SP_EUNSUPPORTED;
  const size_t need = score_ws(G, SP_SCORE_FUSED);
  if (ws == nullptr || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return SP_EWORKSPACE;
  return from_cuda(fused_score_acc(reinterpret_cast<const __nv_bfloat16*>(Q), reinterpret_cast<const __nv_bfloat16*>(K),
                                   G, Lay, acc2, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream)));
}

sp_status sp_acc_importance(const float* acc2, int32_t B, int32_t R_valid, int64_t N, float* importance,
                            sp_stream stream) {
  if (acc2 == nullptr || importance == nullptr || B < 1 || R_valid < 1 || N < 1) return SP_EINVAL;
  sp_status s = check_device();
  if (s != SP_OK) return s;
  return from_cuda(acc_importance(acc2, B, R_valid, N, importance, reinterpret_cast<cudaStream_t>(stream)));
}

size_t sp_score_peer_buffer_bytes(const sp_geom* g, int32_t world, int32_t sm_budget) {
  if (check_geom(g) != SP_OK || world < 1 || world > 8) return 0;
  return fused_peer_buffer_bytes(to_geom(*g), world, sm_budget);
}

size_t sp_score_peer_workspace_bytes(const sp_geom* g, int32_t world, int32_t sm_budget) {
  if (check_geom(g) != SP_OK) return 0;
  if (world < 1 || world > 8) return 0;
  return fused_peer_ws_bytes(to_geom(*g), world, sm_budget);
}

sp_status sp_score_peer_plan(const sp_geom* g, int32_t world, int32_t sm_budget, int64_t out[10]) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if (out == nullptr || world < 1 || world > 8) return SP_EINVAL;
  long long o[kPlanInfo];
  if (!fused_peer_plan_info(to_geom(*g), world, sm_budget, o)) return SP_EUNSUPPORTED;
  for (int i = 0; i < kPlanInfo; ++i) out[i] = o[i];
  return SP_OK;
}

sp_status sp_score_peer(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, int32_t rank,
                        int32_t world, void* const* peer_buffers, int32_t sm_budget, float* importance, void* ws,
                        size_t ws_bytes, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if (importance == nullptr || world < 1 || world > 8 || rank < 0 || rank >= world || sm_budget < 0) return SP_EINVAL;
  if (world > 1 && peer_buffers == nullptr) return SP_EINVAL;
  if (world > 1)
    for (int r = 0; r < world; ++r)
      if (peer_buffers[r] == nullptr || (reinterpret_cast<uintptr_t>(peer_buffers[r]) & 255u) != 0) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  const Geom G = to_geom(*g);
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q, K)) return SP_EUNSUPPORTED;
  const size_t need = fused_peer_ws_bytes(G, world, sm_budget);
  if (need == 0) return SP_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return SP_EWORKSPACE;
  return from_cuda(fused_score_peer(reinterpret_cast<const __nv_bfloat16*>(Q),
                                    reinterpret_cast<const __nv_bfloat16*>(K), G, Lay, rank, world, peer_buffers,
                                    sm_budget, importance, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream)));
}

// Row f4: e4m3 inputs.  The per-tensor dequantisation scales fold into the
// softmax scale (s = scale * q_scale * k_scale * <Q8, K8>, one fp32 product).
static sp_status e4m3_geom(const sp_geom* g, float q_scale, float k_scale, Geom* out) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if (!(std::isfinite(q_scale) && q_scale > 0.f && std::isfinite(k_scale) && k_scale > 0.f)) return SP_EINVAL;
  if (g->d % 32 != 0) return SP_EUNSUPPORTED;                    // 32-byte swizzle rows at 1 byte per element
  Geom G = to_geom(*g);
  G.esz = 1;
  G.scale = g->scale * q_scale * k_scale;
  if (!(std::isfinite(G.scale) && G.scale > 0.f)) return SP_EINVAL;
  *out = G;
  return SP_OK;
}

size_t sp_score_e4m3_workspace_bytes(const sp_geom* g) {
  Geom G;
  if (e4m3_geom(g, 1.f, 1.f, &G) != SP_OK) return 0;
  return fused_supported(G, Layout{}, nullptr, nullptr) ? fused_score_ws_bytes(G) : 0;
}

sp_status sp_score_e4m3_plan(const sp_geom* g, int64_t out[10]) {
  Geom G;
  sp_status s = e4m3_geom(g, 1.f, 1.f, &G);
  if (s != SP_OK) return s;
  if (out == nullptr) return SP_EINVAL;
  long long o[kPlanInfo];
  if (!fused_plan_info(G, o)) return SP_EUNSUPPORTED;
  for (int i = 0; i < kPlanInfo; ++i) out[i] = o[i];
  return SP_OK;
}

sp_status sp_score_e4m3(const void* Q8, const void* K8, float q_scale, float k_scale, const sp_geom* g,
                        const sp_layout* lay, float* importance, void* ws, size_t ws_bytes, sp_stream stream) {
  Geom G;
  sp_status s = e4m3_geom(g, q_scale, k_scale, &G);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q8, K8, 1)) != SP_OK) return s;
  if (importance == nullptr) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q8, K8)) return SP_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < fused_score_ws_bytes(G) || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0)
    return SP_EWORKSPACE;
  // the fused kernel takes the element type from G.esz; the pointer type is nominal
  return from_cuda(fused_score(reinterpret_cast<const __nv_bfloat16*>(Q8), reinterpret_cast<const __nv_bfloat16*>(K8),
                               G, Lay, importance, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream)));
}

// Row f4, reading Z2': the look-ahead tokens' keys join each row's softmax denominator.
size_t sp_score_lookahead_workspace_bytes(const sp_geom* g) {
  if (check_geom(g) != SP_OK) return 0;
  const Geom G = to_geom(*g);
  return fused_supported(G, Layout{}, nullptr, nullptr) ? fused_la_ws_bytes(G) : 0;
}

sp_status sp_score_lookahead(const void* Q, const void* K, const sp_lookahead_k* la, const sp_geom* g,
                             const sp_layout* lay, float* importance, void* ws, size_t ws_bytes, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if (la == nullptr || la->K_la == nullptr || importance == nullptr) return SP_EINVAL;
  if ((reinterpret_cast<uintptr_t>(la->K_la) & 1u) != 0) return SP_EINVAL;
  if (la->s_b < 0 || la->s_l < 0 || la->s_g < 0 || la->s_j < 0 || (la->la_shift != 0 && la->la_shift != 1))
    return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  const Geom G = to_geom(*g);
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q, K)) return SP_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < fused_la_ws_bytes(G) || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0)
    return SP_EWORKSPACE;
  LookaheadK lk;
  lk.K = la->K_la;
  lk.s_b = la->s_b; lk.s_l = la->s_l; lk.s_g = la->s_g; lk.s_j = la->s_j;
  lk.shift = la->la_shift;
  return from_cuda(fused_score_la(reinterpret_cast<const __nv_bfloat16*>(Q), reinterpret_cast<const __nv_bfloat16*>(K),
                                  lk, G, Lay, importance, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream)));
}

// Row f3: paged K cache + block table (+ per-request lengths).
size_t sp_score_paged_workspace_bytes(const sp_geom* g) {
  if (check_geom(g) != SP_OK) return 0;
  const Geom G = to_geom(*g);
  return fused_supported(G, Layout{}, nullptr, nullptr) ? fused_score_ws_bytes(G) : 0;
}

// esz = 1: e4m3 codes with the dequantisation scales folded into the softmax scale (row f4)
static sp_status score_paged_impl(const void* Q, const sp_paged_k* K, const sp_geom* g, const sp_layout* lay,
                                  float* importance, void* ws, size_t ws_bytes, sp_stream stream, int esz,
                                  float q_scale, float k_scale) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  Geom G = to_geom(*g);
  if (esz == 1 && (s = e4m3_geom(g, q_scale, k_scale, &G)) != SP_OK) return s;
  if (K == nullptr || importance == nullptr || lay == nullptr) return SP_EINVAL;
  if (K->cache == nullptr || K->block_table == nullptr || (reinterpret_cast<uintptr_t>(K->cache) & 15u) != 0)
    return SP_EINVAL;
  const int bs = K->block_size;
  if (bs < 8 || (bs & (bs - 1)) != 0) return SP_EINVAL;            // a power of two >= 8
  if (K->num_blocks < 1 || K->max_blocks < (g->N + bs - 1) / bs) return SP_EINVAL;
  const long long ks[4] = {K->s_l, K->s_blk, K->s_tok, K->s_g};
  const long long kn[4] = {g->L, K->num_blocks, bs, g->Hkv};
  for (int i = 0; i < 4; ++i) {
    if (ks[i] < 0) return SP_EINVAL;
    if (kn[i] > 1 && (ks[i] * esz) % 16 != 0) return SP_EINVAL;
  }
  // Q strides: reuse the contiguous-layout check with a dummy K view of the same geometry
  sp_layout ql = *lay;
  ql.k_i = g->d;
  ql.k_g = ql.k_i * g->N;
  ql.k_l = ql.k_g * g->Hkv;
  ql.k_b = ql.k_l * g->L;
  if ((s = check_layout(g, &ql, Q, K->cache, esz)) != SP_OK) return s;
  if ((s = check_device()) != SP_OK) return s;
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q, K->cache)) return SP_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < fused_score_ws_bytes(G) || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0)
    return SP_EWORKSPACE;
  PagedK pk;
  pk.cache = K->cache;
  pk.s_l = K->s_l; pk.s_blk = K->s_blk; pk.s_tok = K->s_tok; pk.s_g = K->s_g;
  pk.num_blocks = K->num_blocks; pk.bs = bs;
  pk.btab = K->block_table; pk.max_blocks = K->max_blocks; pk.seq_lens = K->seq_lens;
  return from_cuda(fused_score_paged(reinterpret_cast<const __nv_bfloat16*>(Q), pk, G, Lay, importance, ws, ws_bytes,
                                     reinterpret_cast<cudaStream_t>(stream)));
}

sp_status sp_score_paged(const void* Q, const sp_paged_k* K, const sp_geom* g, const sp_layout* lay,
                         float* importance, void* ws, size_t ws_bytes, sp_stream stream) {
  return score_paged_impl(Q, K, g, lay, importance, ws, ws_bytes, stream, 2, 1.f, 1.f);
}

sp_status sp_score_paged_e4m3(const void* Q8, const sp_paged_k* K, float q_scale, float k_scale, const sp_geom* g,
                              const sp_layout* lay, float* importance, void* ws, size_t ws_bytes, sp_stream stream) {
  return score_paged_impl(Q8, K, g, lay, importance, ws, ws_bytes, stream, 1, q_scale, k_scale);
}

sp_status sp_score_tune(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, int64_t out[3],
                        float* ms_per_launch, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if ((s = check_device()) != SP_OK) return s;
  const Geom G = to_geom(*g);
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q, K)) return SP_EUNSUPPORTED;
  int tg = 0, ug = 0, h = 0;
  float ms = 0.f;
  s = from_cuda(fused_tune(reinterpret_cast<const __nv_bfloat16*>(Q), reinterpret_cast<const __nv_bfloat16*>(K), G,
                           Lay, reinterpret_cast<cudaStream_t>(stream), &tg, &ug, &h, &ms));
  if (out != nullptr) { out[0] = tg; out[1] = ug; out[2] = h; }
  if (ms_per_launch != nullptr) *ms_per_launch = ms;
  return s;
}

sp_status sp_score_e4m3_tune(const void* Q8, const void* K8, float q_scale, float k_scale, const sp_geom* g,
                             const sp_layout* lay, int64_t out[3], float* ms_per_launch, sp_stream stream) {
  Geom G;
  sp_status s = e4m3_geom(g, q_scale, k_scale, &G);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q8, K8, 1)) != SP_OK) return s;
  if ((s = check_device()) != SP_OK) return s;
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q8, K8)) return SP_EUNSUPPORTED;
  int tg = 0, ug = 0, h = 0;
  float ms = 0.f;
  s = from_cuda(fused_tune(reinterpret_cast<const __nv_bfloat16*>(Q8), reinterpret_cast<const __nv_bfloat16*>(K8), G,
                           Lay, reinterpret_cast<cudaStream_t>(stream), &tg, &ug, &h, &ms));
  if (out != nullptr) { out[0] = tg; out[1] = ug; out[2] = h; }
  if (ms_per_launch != nullptr) *ms_per_launch = ms;
  return s;
}

sp_status sp_score_set_plan(const sp_geom* g, int32_t n_tg, int32_t n_ug, int32_t hier) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if (n_tg > 0 && (n_ug < 1 || hier < 0 || hier > 1)) return SP_EINVAL;
  fused_set_plan(to_geom(*g), n_tg, n_ug, hier);
  return SP_OK;
}

sp_status sp_score_plan(const sp_geom* g, int64_t out[10]) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if (out == nullptr) return SP_EINVAL;
  long long o[kPlanInfo];
  if (!fused_plan_info(to_geom(*g), o)) return SP_EUNSUPPORTED;
  for (int i = 0; i < kPlanInfo; ++i) out[i] = o[i];
  return SP_OK;
}

sp_status sp_trace_enable(uint64_t* device_buffer, int64_t records) {
  if (device_buffer == nullptr || records < 8) {
    fused_set_trace(nullptr, 0);
    return SP_OK;
  }
  fused_set_trace(reinterpret_cast<unsigned long long*>(device_buffer), records);
  return SP_OK;
}

// The split API runs the fused tensor-core kernel in its stats-only / finish-only
// modes when the geometry is supported (SP_SPLIT_ALGO=simt forces the SIMT pair).
bool split_fused(const Geom& g) {
  const char* e = std::getenv("SP_SPLIT_ALGO");
  if (e && std::strcmp(e, "simt") == 0) return false;
  return fused_supported(g, Layout{}, nullptr, nullptr);
}

size_t sp_score_split_workspace_bytes(const sp_geom* g) {
  if (check_geom(g) != SP_OK) return 0;
  Geom G = to_geom(*g);
  if (split_fused(G)) return fused_score_ws_bytes(G);
  size_t a = simt_split_ws_bytes(G);
  size_t b = align256((size_t)G.B * G.Rv * G.N * sizeof(unsigned));
  return a > b ? a : b;
}

sp_status sp_score_stats(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, float* stats, void* ws,
                         size_t ws_bytes, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if (stats == nullptr) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  if (ws == nullptr || ws_bytes < sp_score_split_workspace_bytes(g)) return SP_EWORKSPACE;
  const Geom G = to_geom(*g);
  const auto* q = reinterpret_cast<const __nv_bfloat16*>(Q);
  const auto* k = reinterpret_cast<const __nv_bfloat16*>(K);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (split_fused(G)) return from_cuda(fused_score_stats(q, k, G, to_layout(*lay), stats, ws, ws_bytes, st));
  return from_cuda(simt_score_stats(q, k, G, to_layout(*lay), stats, ws, st));
}

sp_status sp_stats_combine(const float* parts, int32_t P, int64_t n_rows, float* lse2, sp_stream stream) {
  if (parts == nullptr || lse2 == nullptr || P < 1 || n_rows < 1) return SP_EINVAL;
  sp_status s = check_device();
  if (s != SP_OK) return s;
  return from_cuda(stats_combine(parts, P, n_rows, lse2, reinterpret_cast<cudaStream_t>(stream)));
}

sp_status sp_score_finish(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, const float* lse2,
                          float* importance, void* ws, size_t ws_bytes, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if (lse2 == nullptr || importance == nullptr) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  if (ws == nullptr || ws_bytes < sp_score_split_workspace_bytes(g)) return SP_EWORKSPACE;
  const Geom G = to_geom(*g);
  const auto* q = reinterpret_cast<const __nv_bfloat16*>(Q);
  const auto* k = reinterpret_cast<const __nv_bfloat16*>(K);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (split_fused(G))
    return from_cuda(fused_score_finish(q, k, G, to_layout(*lay), lse2, importance, ws, ws_bytes, st));
  return from_cuda(simt_score_finish(q, k, G, to_layout(*lay), lse2, importance, ws, st));
}

size_t sp_select_workspace_bytes(int32_t B, int64_t N, const sp_select_params* p) {
  if (check_select(B, N, p) != SP_OK) return 0;
  return select_ws_bytes(B, N, p->chunk);
}

sp_status sp_select(const float* importance, int32_t B, int64_t N, const sp_select_params* p, int32_t* ids,
                    int32_t* pos, int32_t* n_kept, void* ws, size_t ws_bytes, sp_stream stream) {
  return sp_select_gather(importance, nullptr, B, N, p, ids, pos, n_kept, nullptr, ws, ws_bytes, stream);
}

sp_status sp_select_gather(const float* importance, const int32_t* tokens, int32_t B, int64_t N,
                           const sp_select_params* p, int32_t* ids, int32_t* pos, int32_t* n_kept,
                           int32_t* out_tokens, void* ws, size_t ws_bytes, sp_stream stream) {
  sp_status s = check_select(B, N, p);
  if (s != SP_OK) return s;
  if (importance == nullptr || ids == nullptr || pos == nullptr || n_kept == nullptr) return SP_EINVAL;
  if ((tokens == nullptr) != (out_tokens == nullptr)) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  if (ws == nullptr || ws_bytes < select_ws_bytes(B, N, p->chunk)) return SP_EWORKSPACE;
  return from_cuda(select_launch(importance, B, N, p->pool_k, p->chunk, p->pos0, keep_ppm(p->keep_rate), ids, pos,
                                 n_kept, ws, reinterpret_cast<cudaStream_t>(stream), tokens, out_tokens));
}

sp_status sp_select_ragged(const float* importance, const int32_t* seq_lens, const int32_t* tokens, int32_t B,
                           int64_t N, const sp_select_params* p, int32_t* ids, int32_t* pos, int32_t* n_kept,
                           int32_t* out_tokens, void* ws, size_t ws_bytes, sp_stream stream) {
  sp_status s = check_select(B, N, p);
  if (s != SP_OK) return s;
  if (importance == nullptr || seq_lens == nullptr || ids == nullptr || pos == nullptr || n_kept == nullptr)
    return SP_EINVAL;
  if ((tokens == nullptr) != (out_tokens == nullptr)) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  if (ws == nullptr || ws_bytes < select_ws_bytes(B, N, p->chunk)) return SP_EWORKSPACE;
  return from_cuda(select_launch(importance, B, N, p->pool_k, p->chunk, p->pos0, keep_ppm(p->keep_rate), ids, pos,
                                 n_kept, ws, reinterpret_cast<cudaStream_t>(stream), tokens, out_tokens, seq_lens));
}

namespace {
sp_status check_seq(int32_t B, int64_t N, int32_t world, const sp_select_params* p) {
  sp_status s = check_select(B, N, p);
  if (s != SP_OK) return s;
  if (world < 1 || N % world != 0) return SP_EINVAL;
  const int64_t n = N / world;
  if (n % p->chunk != 0 || (p->pool_k - 1) / 2 > n) return SP_EINVAL;
  return SP_OK;
}
}  // namespace

int64_t sp_seq_candidate_count(int64_t N, int32_t world, const sp_select_params* p) {
  if (check_seq(1, N, world, p) != SP_OK) return -1;
  return seq_candidate_count(N, world, p->chunk, keep_ppm(p->keep_rate));
}

size_t sp_seq_select_workspace_bytes(int32_t B, int64_t N, int32_t world, const sp_select_params* p) {
  if (check_seq(B, N, world, p) != SP_OK) return 0;
  return seq_select_ws_bytes(B, N, world, p->chunk);
}

sp_status sp_seq_edges(const float* imp_local, int32_t B, int64_t N, int32_t world, const sp_select_params* p,
                       float* edges, sp_stream stream) {
  sp_status s = check_seq(B, N, world, p);
  if (s != SP_OK) return s;
  if (imp_local == nullptr || (edges == nullptr && p->pool_k > 1)) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  return from_cuda(seq_edges_launch(imp_local, B, N / world, p->pool_k, edges, reinterpret_cast<cudaStream_t>(stream)));
}

sp_status sp_seq_candidates(const float* imp_local, const float* edges_all, int32_t rank, int32_t world, int32_t B,
                            int64_t N, const sp_select_params* p, uint64_t* cand, void* ws, size_t ws_bytes,
                            sp_stream stream) {
  sp_status s = check_seq(B, N, world, p);
  if (s != SP_OK) return s;
  if (rank < 0 || rank >= world || imp_local == nullptr || cand == nullptr) return SP_EINVAL;
  if (edges_all == nullptr && p->pool_k > 1 && world > 1) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  if (ws == nullptr || ws_bytes < seq_select_ws_bytes(B, N, world, p->chunk)) return SP_EWORKSPACE;
  const long long M = seq_candidate_count(N, world, p->chunk, keep_ppm(p->keep_rate));
  return from_cuda(seq_candidates_launch(imp_local, edges_all, rank, world, B, N, p->pool_k, p->chunk, M,
                                         reinterpret_cast<unsigned long long*>(cand), ws,
                                         reinterpret_cast<cudaStream_t>(stream)));
}

sp_status sp_seq_merge(const uint64_t* cand_all, int32_t world, int32_t B, int64_t N, const sp_select_params* p,
                       const int32_t* tokens, int32_t* ids, int32_t* pos, int32_t* n_kept, int32_t* out_tokens,
                       void* ws, size_t ws_bytes, sp_stream stream) {
  sp_status s = check_seq(B, N, world, p);
  if (s != SP_OK) return s;
  if (cand_all == nullptr || ids == nullptr || pos == nullptr || n_kept == nullptr) return SP_EINVAL;
  if ((tokens == nullptr) != (out_tokens == nullptr)) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  if (ws == nullptr || ws_bytes < seq_select_ws_bytes(B, N, world, p->chunk)) return SP_EWORKSPACE;
  const long long ppm = keep_ppm(p->keep_rate);
  const long long M = seq_candidate_count(N, world, p->chunk, ppm);
  return from_cuda(seq_merge_launch(reinterpret_cast<const unsigned long long*>(cand_all), world, B, N, p->pool_k,
                                    p->chunk, p->pos0, ppm, M, tokens, ids, pos, n_kept, out_tokens, ws,
                                    reinterpret_cast<cudaStream_t>(stream)));
}

sp_status sp_gather(const int32_t* tokens, const int32_t* ids, const int32_t* n_kept, int32_t B, int64_t N,
                    int32_t* out, sp_stream stream) {
  if (tokens == nullptr || ids == nullptr || n_kept == nullptr || out == nullptr || B < 1 || N < 1 ||
      N >= (1LL << 31))
    return SP_EINVAL;
  sp_status s = check_device();
  if (s != SP_OK) return s;
  return from_cuda(gather_launch(tokens, ids, n_kept, B, N, out, reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"

namespace {
// The whole device path (validated arguments; ws = score workspace, then the
// selection's): when the fused kernel can stage them, the selection's phase A
// (pooling + chunk means) runs in the score kernel's epilogue and the selection
// launch -- a programmatic dependent -- does phases B-C only; otherwise the
// score, then the full selection (+ gather).  Same bits either way.
// smallest number of unit groups per token group for which the deferred finalize
// pays (SP_DEFER_MIN_UG overrides: A/B timing)
int defer_min_ug() {
  const char* e = std::getenv("SP_DEFER_MIN_UG");
  return e ? std::atoi(e) : 2;
}

sp_status score_select_dev(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay,
                           const sp_select_params* p, const int32_t* tokens, float* importance, int32_t* ids,
                           int32_t* pos, int32_t* n_kept, int32_t* out_tokens, void* ws, size_t ws_bytes,
                           sp_stream stream) {
  const Geom G = to_geom(*g);
  const Layout Lay = to_layout(*lay);
  const size_t sb = align256(score_ws(G, SP_SCORE_AUTO));
  void* sws = reinterpret_cast<char*>(ws) + sb;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  long long plan[kPlanInfo] = {};
  const int kDeferMinUg = defer_min_ug();
  const bool epilogue_ab = std::getenv("SP_SELECT_EPILOGUE") != nullptr;   // A/B knob (timing, tests)
  if (!epilogue_ab && resolve_algo(G, SP_SCORE_AUTO) == SP_SCORE_FUSED && fused_supported(G, Lay, Q, K) &&
      fused_plan_info(G, plan) && plan[3] >= kDeferMinUg &&
      select_deferred_supported(g->N, g->R_valid, (int)plan[3], p->pool_k, p->chunk)) {
    // the score kernel without its cross-unit-group epilogue; the selection
    // finalizes the importance from the partial maps (same bits).  Measured
    // (DESIGN.md 5.3): C1 step -4 us, C3 -5 us, C2 and C4 even or better
    const float* accp = nullptr;
    int n_ug = 0;
    long long pitch = 0;
    const cudaError_t e = fused_score_deferred(reinterpret_cast<const __nv_bfloat16*>(Q),
                                               reinterpret_cast<const __nv_bfloat16*>(K), G, Lay, ws, sb, st, &accp,
                                               &n_ug, &pitch);
    if (e == cudaSuccess)
      return from_cuda(select_deferred_launch(accp, pitch, n_ug, g->R_valid, importance, g->B, g->N, p->pool_k, p->chunk,
                                              p->pos0, keep_ppm(p->keep_rate), ids, pos, n_kept, sws, st, tokens,
                                              out_tokens));
    if (e != cudaErrorNotSupported) return from_cuda(e);
  }
  if (epilogue_ab && resolve_algo(G, SP_SCORE_AUTO) == SP_SCORE_FUSED &&
      fused_supported(G, Lay, Q, K)) {                 // A/B: the chunk means in the score kernel's epilogue
    const ChunkOut co{select_ws_scores(sws, g->B), p->pool_k, p->chunk};
    const cudaError_t e = fused_score_chunks(reinterpret_cast<const __nv_bfloat16*>(Q),
                                             reinterpret_cast<const __nv_bfloat16*>(K), G, Lay, importance, co, ws, sb,
                                             st);
    if (e == cudaSuccess)
      return from_cuda(select_ready_launch(g->B, g->N, p->chunk, keep_ppm(p->keep_rate), p->pos0, ids, pos, n_kept,
                                           sws, st, tokens, out_tokens));
    if (e != cudaErrorNotSupported) return from_cuda(e);
  }
  sp_status s = sp_score(Q, K, g, lay, importance, ws, sb, stream);
  if (s != SP_OK) return s;
  return sp_select_gather(importance, tokens, g->B, g->N, p, ids, pos, n_kept, out_tokens, sws, ws_bytes - sb, stream);
}
}  // namespace

extern "C" {

size_t sp_score_select_workspace_bytes(const sp_geom* g, const sp_select_params* p) {
  if (check_geom(g) != SP_OK || check_select(g->B, g->N, p) != SP_OK) return 0;
  return align256(score_ws(to_geom(*g), SP_SCORE_AUTO)) + select_ws_bytes(g->B, g->N, p->chunk);
}

sp_status sp_score_select(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay,
                          const sp_select_params* p, const int32_t* tokens, float* importance, int32_t* ids,
                          int32_t* pos, int32_t* n_kept, int32_t* out_tokens, void* ws, size_t ws_bytes,
                          sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if ((s = check_select(g->B, g->N, p)) != SP_OK) return s;
  if (importance == nullptr || ids == nullptr || pos == nullptr || n_kept == nullptr) return SP_EINVAL;
  if ((tokens == nullptr) != (out_tokens == nullptr)) return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  if (ws == nullptr || ws_bytes < sp_score_select_workspace_bytes(g, p) || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0)
    return SP_EWORKSPACE;
  return score_select_dev(Q, K, g, lay, p, tokens, importance, ids, pos, n_kept, out_tokens, ws, ws_bytes, stream);
}

sp_status sp_score_chunks(const void* Q, const void* K, const sp_geom* g, const sp_layout* lay, int32_t pool_k,
                          int32_t chunk, float* importance, float* cs, void* ws, size_t ws_bytes, sp_stream stream) {
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, Q, K)) != SP_OK) return s;
  if (importance == nullptr || cs == nullptr || pool_k < 1 || pool_k % 2 == 0 || chunk < 1) return SP_EINVAL;
  if (!select_supported(pool_k) || chunk > 16384) return SP_EUNSUPPORTED;
  if ((s = check_device()) != SP_OK) return s;
  const Geom G = to_geom(*g);
  const Layout Lay = to_layout(*lay);
  if (!fused_supported(G, Lay, Q, K)) return SP_EUNSUPPORTED;
  const size_t need = score_ws(G, SP_SCORE_FUSED);
  if (ws == nullptr || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return SP_EWORKSPACE;
  const ChunkOut co{cs, pool_k, chunk};
  const cudaError_t e = fused_score_chunks(reinterpret_cast<const __nv_bfloat16*>(Q),
                                           reinterpret_cast<const __nv_bfloat16*>(K), G, Lay, importance, co, ws,
                                           ws_bytes, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaErrorNotSupported ? SP_EUNSUPPORTED : from_cuda(e);
}

size_t sp_run_workspace_bytes(const sp_geom* g, const sp_select_params* p) {
  if (check_geom(g) != SP_OK || check_select(g->B, g->N, p) != SP_OK) return 0;
  // score and select get disjoint regions: the fused score kernel's counters
  // must stay zero between calls
  return align256(score_ws(to_geom(*g), SP_SCORE_AUTO)) + select_ws_bytes(g->B, g->N, p->chunk);
}

sp_status sp_run_host(const sp_host_io* host, const sp_device_bufs* dev, const sp_geom* g, const sp_layout* lay,
                      const sp_select_params* p, sp_stream stream) {
  if (host == nullptr || dev == nullptr) return SP_EINVAL;
  if (host->Q == nullptr || host->K == nullptr || host->tokens == nullptr || host->ids == nullptr ||
      host->pos == nullptr || host->n_kept == nullptr || host->out_tokens == nullptr)
    return SP_EINVAL;
  sp_status s = check_geom(g);
  if (s != SP_OK) return s;
  if ((s = check_layout(g, lay, dev->Q, dev->K)) != SP_OK) return s;
  if ((s = check_select(g->B, g->N, p)) != SP_OK) return s;
  if (dev->ws == nullptr || dev->ws_bytes < sp_run_workspace_bytes(g, p) ||
      (reinterpret_cast<uintptr_t>(dev->ws) & 255u) != 0)
    return SP_EWORKSPACE;
  if (dev->importance == nullptr || dev->ids == nullptr || dev->pos == nullptr || dev->n_kept == nullptr ||
      dev->tokens == nullptr || dev->out_tokens == nullptr)
    return SP_EINVAL;
  if ((s = check_device()) != SP_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t tok_bytes = (size_t)g->B * g->N * sizeof(int32_t);
  if (cudaMemcpyAsync(dev->Q, host->Q, host->q_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(dev->K, host->K, host->k_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(dev->tokens, host->tokens, tok_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaGetLastError();
    return SP_ECUDA;
  }
  if ((s = score_select_dev(dev->Q, dev->K, g, lay, p, dev->tokens, dev->importance, dev->ids, dev->pos, dev->n_kept,
                            dev->out_tokens, dev->ws, dev->ws_bytes, stream)) != SP_OK)
    return s;
  if (cudaMemcpyAsync(host->n_kept, dev->n_kept, (size_t)g->B * sizeof(int32_t), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(host->ids, dev->ids, tok_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(host->pos, dev->pos, tok_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(host->out_tokens, dev->out_tokens, tok_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess) {
    cudaGetLastError();
    return SP_ECUDA;
  }
  return SP_OK;
}

}  // extern "C"
