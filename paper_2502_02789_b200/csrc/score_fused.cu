// Fused token-importance kernel for sm_100a: one HBM read of K.
//
// Computes, for every request b and prompt token i (O1-O4;
// PAPER.md sec:token_importance eq. P:105-107 and sec:attn_agg P:119):
//   x[l,h,r,i]  = scale*log2(e) * <Q[b][l][r][h], K[b][l][h/G][i]>   (log2-domain logit)
//   lse2[l,h,r] = log2 sum_i 2^x[l,h,r,i]            (softmax over the N prompt keys, Z2)
//   acc[r,i]    = max_{l,h} (x - lse2)               (max over H and L, log domain)
//   imp[b][i]   = (1/Rv) sum_{r<Rv} 2^acc[r,i]       (mean over the valid look-ahead rows)
//
// Design:
// * Persistent cooperative grid, one CTA per SM.  A request's N tokens are cut
//   into 128-token tiles and its L*Hkv (layer, kv-head) "units" into groups; a
//   job = (request, token group, unit group).  All jobs of one request run in
//   the same wave of CTAs, so every CTA that shares a unit is co-resident.
// * Warp roles (384 threads): warp 0 TMA producer, warp 1 tcgen05.mma issuer
//   (+TMEM owner), warp 2 statistics exchange, warp 3 lse2 gather (and, when
//   the prompt is sequence-sharded over GPUs, the cross-rank merge), warps 4-7
//   softmax statistics, warps 8-11 max-aggregation.  The TMA/MMA warps run warp-uniform loops and
//   issue from one elected lane.
// * K tiles [128 tokens x d] bf16 stream HBM -> SMEM by TMA (swizzled); the
//   unit's query block [G*Rv x d] is the MMA B operand; each tile's logits
//   D[128 x NCP] fp32 go to the next slot of a 16-slot TMEM ring and stay
//   there until aggregated: logits never leave the chip, K is read once.
// * Statistics warps fold every tile into per-column running sums as soon as
//   its MMA lands; the exchange warp publishes the CTA partial (one 64-bit
//   (max, sum) word per column); the gather warp polls the unit's partials of
//   all token groups and merges them in fixed order (bit-identical lse2 in
//   every CTA); the aggregation warps fold max_h (x - lse2) into a per-token
//   running max in SMEM and release the TMEM slots.
// * Cross-unit-group max: partial acc maps go to the workspace and the CTAs of
//   a token group split the final mean-of-exp2 among themselves.
// * Instantiated per GQA group size and per "one 32-column group" (NCP = 32):
//   the warp roles share the SM's instruction cache, so the executed code is
//   kept small (measured: code size moved C3 by > 20 %).
#include "sp_internal.h"

#include <cuda.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

namespace sp {
namespace {

constexpr int kThreads = 384;
// Timeline tracing (sp_trace_enable) is compiled in only with -DSP_FUSED_TRACE
// (tools/ab_build.sh ... -DSP_FUSED_TRACE): the product kernel carries no
// trace code (the warp roles share the SM's instruction cache).
#ifdef SP_FUSED_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif
enum FusedMode : int { kModeFull = 0, kModeStats = 1, kModeFinish = 2 };
constexpr int kTileM = 128;
constexpr int kStatsWarp0 = 4;
constexpr int kFinalWarp0 = 8;
constexpr int kMaxStages = 8;
// Stage cap of the plans (measured, r2 tools/gpu_r2_stages.sh, gpu_r2_pst.sh): more
// TMA tiles in flight than 4 slow the bf16 kernel down (C3 37x4: 4 stages 0.3405 ms,
// 5: 0.3442; C1 8x16: 0.0720 vs 0.0745); some geometries prefer 3 (a 16K prompt:
// 0.1916 vs 0.1964 ms; the C4/8 peer shard 0.2122 vs 0.2190), others 4 (C2: 0.641
// vs 0.672 ms), so the tuner tries both; peer plans (no tuner) take 3.  The e4m3
// kernel is indifferent (3..8 stages within 0.5 %).
constexpr int kStageCap = 4;
constexpr int kStageCapPeer = 3;
constexpr int kMaxChunks = 8;          // NCP <= 128 columns (16-column chunks)
constexpr int kMaxSlots = 16;          // TMEM tile slots (512 columns / 32)
constexpr int kLseRing = 8;            // lse2 buffers in SMEM (gather may run ahead of aggregation)
constexpr int kMaxQSlots = 4;          // query blocks in SMEM (the producer loads up to nq - 1 units ahead)
constexpr int kMaxLseBatch = 10;       // 64-bit partial words in flight per lane
constexpr int kMaxPeers = 8;           // ranks of a peer-memory statistics exchange
constexpr int kTmemCols = 512;
constexpr double kSmHbmBytesPerUs = 7.0e6 / 148;   // one SM's share of ~7 TB/s, bytes per microsecond
constexpr int kSmemLimit = 232448;     // sm_100 max dynamic shared memory per block

// ------------------------------------------------------------------ parameters
struct FusedParams {
  CUtensorMap tmK;                     // 5-D: {d, N, Hkv, L, B}
  CUtensorMap tmQ;                     // 5-D: {d, H, R, L, B}
  int B, L, Hkv, G, Rv, d, N;
  int T, U;                            // tiles / units per request
  int n_tg, n_ug, J;                   // token groups, unit groups, jobs per request
  long long total_jobs;
  int NC, NCP, W, nkb, stages, nslots, tpc;
  int esz, swb, ksteps;                // element bytes (2 bf16, 1 e4m3), swizzle-block bytes, K steps per block
  float xs;                            // scale * log2(e)
  uint32_t idesc;                      // tcgen05 instruction descriptor
  uint32_t layout_type;                // UMMA smem descriptor swizzle code
  // smem carve (byte offsets from the 1024-aligned base)
  uint32_t off_k, off_q, off_acc, off_red, off_lse, off_comb, off_bar, off_bt;
  uint32_t k_stage_bytes, q_slot_bytes;
  int nq;                              // query slots (2 or 4, power of two)
  // row f3: paged K (tmK is then 5-D {d, Hkv, block_size, blocks, L}) and per-request lengths
  int paged, bs, bs_log2;              // paged: 1; tokens per block (a power of two >= 8), its log2
  int kinter, fl, fb;                  // kb-interleaved tiles (one box per block): idx = l*fl + blk*fb + g
  const int* btab;                     // [B][max_blocks] physical block ids
  int max_blocks;
  const int* seq_lens;                 // [B] prompt lengths in [1, N] (clamped), or null: all N
  const float2* la;                    // Z2' (row f4): [B][U][NCP] look-ahead keys' (max2, sum) per column, or null
  // workspace
  unsigned long long* part;            // [2][B][U][n_tg][NCP] CTA partials, one buffer per launch parity:
                                       // (max2, sum) packed in one 64-bit word; 0 = "not yet written"
  int hier;                            // cross-rank (peer) exchange: world > 1
  unsigned* epoch;                     // [2] launch epoch (parity selects the partial buffer), CTAs done
  float* accpart;                      // [B][n_ug][Rv][acc_pitch] the unit groups' partial (l,h)-max maps
  long long acc_pitch;                 // row pitch of accpart in floats: N rounded to 32, + 32 (rows that are a
                                       // power-of-two apart camp on the same L2 slices)
  unsigned* fin_cnt;                   // [3][B][n_tg] finalize counters: [launch parity] in the full and
                                       // statistics modes (the other parity's re-zeroed by the exchange
                                       // warp), [2] in finish mode (self-resetting: a second count)
  float* imp;                          // [B][N]
  float* acc_out;                      // head-sharded partition: [B][Rv][N] log2-domain max instead of imp
  int* err;
  unsigned long long* trace;           // optional [grid][trace_units][8] globaltimer stamps (debug)
  int trace_units;
  unsigned long long* tile_trace;      // optional [1000][8] per-tile MMA stamps of CTA 0 (debug)
  int mode;                            // kModeFull / kModeStats (publish partials only) / kModeFinish (lse2 given)
  const float* lse_in;                 // kModeFinish: lse2 per row ((b*L + l)*H + h)*Rv + r
  // peer-memory exchange (sequence-sharded single pass, world > 1): world ranks
  // each score their own tokens; every CTA merges its rank's n_tg partials into
  // the rank word, the unit's designated CTA (token group u mod n_tg) stores it
  // into row `rank` of every peer's rank-word buffer, and every CTA merges the
  // unit's `world` rank words in rank order (the same lse2 bits on every rank;
  // peer_merge_col).
  int rank, world;
  unsigned long long* peer[kMaxPeers]; // every rank's rank-word buffer base ([2][B][U][world][NCP])
  int l2hint;                          // K tiles loaded with an L2 evict_first hint (plan; A/B: SP_FUSED_L2HINT)
  // selection phase A in the epilogue (sp_score_select): chunk means of every
  // token group, written into the selection workspace (null: importance only)
  float* cs_out;                       // [B][n_c_row] chunk scores
  unsigned* bnd_cnt;                   // [B][n_tg] token-group boundary counters (self-resetting)
  int pool_k, chunk;
  long long n_c_row;
  int defer;                           // sp_score_select: the unit groups' partial maps are the output, the
                                       // selection launch finalizes the importance (no cross-CTA epilogue)
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// The TMA / MMA helpers below are called by a whole (converged) warp and issue
// from one elected lane: the loop state stays warp-uniform, so descriptors and
// coordinates live in uniform registers (no per-instruction R2UR + elect loop).
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(bar),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe of an mbarrier phase (no suspend): the cheap fast path.
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Wait for an mbarrier phase.  After a few immediate retries the waiting warp
// backs off with __nanosleep so that idle waiters (up to half the CTA's warps at
// any time) do not steal issue slots from the epilogue warps on their SMSP.
// Bounded: a pipeline that never completes (a bug) traps after ~4 s.
__device__ __noinline__ void mbar_wait_slow(uint32_t bar, uint32_t parity) {
  uint64_t t0 = 0;
  for (uint32_t i = 1;; ++i) {
    if (mbar_try_wait(bar, parity)) return;
    if (i > 4) __nanosleep(i < 32 ? 20 : 80);
    if ((i & 1023) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) asm volatile("trap;");
    }
  }
}
// Fast path inline (one try_wait); the back-off loop is out of line to keep
// the warp roles' hot code small (they share the SM's instruction cache).
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (!mbar_test_wait(bar, parity)) mbar_wait_slow(bar, parity);
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n\t}" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
// With an L2 cache-policy hint (createpolicy, e.g. evict_first for the K stream).
__device__ __forceinline__ void tma_load_5d_hint(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2, int c3, int c4, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;\n\t}" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "l"(policy)
      : "memory");
}
// Per-lane variant (no election): every calling lane issues its own box.
__device__ __forceinline__ void tma_load_5d_lane(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout_type) {
  uint64_t desc = 0;
  desc |= (uint64_t)((saddr >> 4) & 0x3FFFu);               // [0,14)  start address >> 4
  desc |= (uint64_t)1u << 16;                                // [16,30) LBO (unused for swizzled K-major)
  desc |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;     // [32,46) SBO: 8-row group stride
  desc |= (uint64_t)1u << 46;                                // [46,48) version = 1 (sm_100)
  desc |= (uint64_t)(layout_type & 7u) << 61;                // [61,64) swizzle mode
  return desc;
}
// kF8: kind::f8f6f4 (e4m3 x e4m3, K = 32 per instruction) instead of kind::f16
// (bf16 x bf16, K = 16); both step 32 bytes of a K-major row per instruction.
template <bool kF8>
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (kF8) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}
// One tile's K steps (KS = d*esz/32) with compile-time descriptor offsets;
// KSTEPS 32-byte steps per 128-byte swizzle block.
template <int KS, int KSTEPS, bool kF8>
__device__ __forceinline__ void issue_tile(uint32_t dcol, uint32_t a_lo0, uint32_t b_lo0, uint32_t desc_hi,
                                           uint32_t b_kb, uint32_t idesc) {
#pragma unroll
  for (int j = 0; j < KS; ++j) {
    const uint32_t kb = j / KSTEPS, ks = j % KSTEPS;
    umma<kF8>(dcol, ((uint64_t)desc_hi << 32) | (a_lo0 + kb * (256u * KSTEPS) + ks * 2u),
              ((uint64_t)desc_hi << 32) | (b_lo0 + kb * b_kb + ks * 2u), idesc, j > 0 ? 1u : 0u);
  }
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, float (&v)[16]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tie16(float (&v)[16]) {
  asm volatile(""
               : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]),
                 "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]), "+f"(v[12]), "+f"(v[13]), "+f"(v[14]),
                 "+f"(v[15]));
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long pack_ms(float m, float s) {
  return (unsigned long long)__float_as_uint(m) | ((unsigned long long)__float_as_uint(s) << 32);
}
__device__ __forceinline__ float2 unpack_ms(unsigned long long w) {
  return make_float2(__uint_as_float((unsigned)w), __uint_as_float((unsigned)(w >> 32)));
}

// Shared-memory unsigned max without return (explicitly shared: the pointers
// into the manually aligned SMEM carve are generic to the compiler).
__device__ __forceinline__ void red_smem_max(uint32_t saddr, unsigned v) {
  asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void set_err(int* err, int code) { atomicCAS(err, 0, code); }

// Spin (one thread) until *p >= target; bounded so a broken exchange can never hang the GPU.
// (deadline 2 s of globaltimer: before mbar_wait_slow's 4 s trap)
__device__ __forceinline__ void spin_geq(const unsigned* p, unsigned target, int* err) {
  long long it = 0;
  unsigned long long t_dead = 0;
  while (ld_acquire(p) < target) {
    ++it;
    if ((it & 1023) == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
      if (t_dead == 0) t_dead = now + 2000000000ull;
      else if (now > t_dead) {
        set_err(err, kDevTimeout);
        return;
      }
    }
    if (it > 8) __nanosleep(it < 64 ? 32 : 100);
  }
}


// 2^x with one MUFU op (flush-to-zero: results below 2^-126 contribute nothing
// measurable to a softmax denominator or a probability > 1e-30).
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}


// Debug trace: stamp event e of the CTA's ui-th unit (no-op unless enabled).
__device__ __forceinline__ void trace_stamp(const FusedParams& p, uint32_t ui, int e) {
  if constexpr (!kTrace) return;
  if (p.trace != nullptr && ui < (uint32_t)p.trace_units)
    p.trace[((size_t)blockIdx.x * p.trace_units + ui) * 8 + e] = globaltimer_ns();
}


// Debug wait accounting (trace mode only): mbar_wait plus the time it took.
__device__ __forceinline__ void mbar_wait_acc(const FusedParams& p, uint32_t bar, uint32_t parity,
                                              unsigned long long& acc) {
  if (!kTrace || p.trace == nullptr) { mbar_wait(bar, parity); return; }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  acc += clock64() - t0;
}
__device__ __forceinline__ void trace_waits(const FusedParams& p, int k, unsigned long long v) {
  if constexpr (!kTrace) return;
  if (p.trace != nullptr && p.trace_units > 1)
    p.trace[((size_t)blockIdx.x * p.trace_units + p.trace_units - 1) * 8 + k] = v;
}

// Fold one tile's 32 logit columns (group grp) into the running (l,h)-max of
// this thread's token: acc[(t*Rv + r)*128 + tok] = max(acc, max_h (x*xs - lse2)).
// Columns are r-major (c = r*G + h).  kG > 0: compile-time group size dividing 32.
template <int kG, int kW>
__device__ __forceinline__ void fold_tile(const float (&x)[kW], const float (&lv)[kW], float xs, int grp, int NC,
                                          int G, int Rv, float* arow) {
  if constexpr (kG > 0) {
#pragma unroll
    for (int rr = 0; rr < kW / kG; ++rr) {
      const int r = grp * (kW / kG) + rr;
      if (r < Rv) {
        float best = fmaf(x[rr * kG], xs, -lv[rr * kG]);
#pragma unroll
        for (int h = 1; h < kG; ++h) best = fmaxf(best, fmaf(x[rr * kG + h], xs, -lv[rr * kG + h]));
        float* a = arow + r * kTileM;
        *a = fmaxf(*a, best);
      }
    }
  } else {
    // generic G: rows may straddle column groups; the row index is recomputed
    float best = -CUDART_INF_F;
    int cur = -1;
#pragma unroll
    for (int i = 0; i < kW; ++i) {
      const int c = grp * kW + i;
      if (c < NC) {
        const int r = c / G;
        if (r != cur) {
          if (cur >= 0) {
            float* a = arow + cur * kTileM;
            *a = fmaxf(*a, best);
          }
          best = -CUDART_INF_F;
          cur = r;
        }
        best = fmaxf(best, fmaf(x[i], xs, -lv[i]));
      }
    }
    if (cur >= 0) {
      float* a = arow + cur * kTileM;
      *a = fmaxf(*a, best);
    }
  }
}

struct Job {
  int b, tg, ug, t_lo, t_hi, u_lo, u_hi;
  int n;                                   // this request's prompt tokens (N unless seq_lens)
};
// Out of line: called once per job by every role; its 64-bit divisions would
// otherwise be inlined into each role's code.
__device__ __noinline__ Job decode_job(const FusedParams& p, long long job) {
  Job j;
  j.b = (int)(job / p.J);
  const int r = (int)(job % p.J);
  j.tg = r / p.n_ug;
  j.ug = r % p.n_ug;
  j.n = p.seq_lens ? min(max(p.seq_lens[j.b], 1), p.N) : p.N;
  const int T = p.seq_lens ? (j.n + kTileM - 1) / kTileM : p.T;   // the request's tiles (ragged batch)
  j.t_lo = (int)((long long)j.tg * T / p.n_tg);
  j.t_hi = (int)((long long)(j.tg + 1) * T / p.n_tg);
  j.u_lo = (int)((long long)j.ug * p.U / p.n_ug);
  j.u_hi = (int)((long long)(j.ug + 1) * p.U / p.n_ug);
  return j;
}

// Row f3: one 128-token K tile of request jb.b from a paged cache (block table).
// block_size >= 128: one box of 128 tokens inside one block; block_size < 128:
// 128 / block_size boxes, one per block, each landing at its row offset of the
// tile (block_size >= 8 rows keeps every box on a swizzle-atom boundary).
// Blocks wholly past the request's length are not loaded (their rows are
// masked downstream); expect_tx counts the bytes actually requested.  Out of
// line: the producer's hot loop stays small for the contiguous layout.
// bts: the job's block-table slice in SMEM (entry 0 = the block of token t_lo * 128).
__device__ __noinline__ void paged_tile(const FusedParams& p, uint32_t kdst, uint32_t bar, const Job& jb, int t, int g,
                                        int l, int lane, const int* bts) {
  // (32-bit shifts: the block size is a power of two; token indices < 2^31)
  const int tok0 = t * kTileM;
  const int blk0 = (jb.t_lo * kTileM) >> p.bs_log2;
  if (p.bs >= kTileM) {
    const int blk = bts[(tok0 >> p.bs_log2) - blk0];
    const int off = tok0 & (p.bs - 1);
    mbar_expect_tx(bar, p.k_stage_bytes);
    for (int kb = 0; kb < p.nkb; ++kb) tma_load_5d(kdst + kb * (kTileM * p.swb), &p.tmK, bar, kb * p.W, g, off, blk, l);
  } else {
    // one lane per block: the boxes are issued in parallel
    const int nb = kTileM >> p.bs_log2;
    const int nvalid = min(nb, (jb.n - tok0 + p.bs - 1) >> p.bs_log2);
    mbar_expect_tx(bar, (uint32_t)(nvalid * p.bs * p.swb * p.nkb));
    __syncwarp();
    if (lane < nvalid) {
      const int blk = bts[(tok0 >> p.bs_log2) - blk0 + lane];
      if (p.kinter)                                                     // the whole block row span in one box
        tma_load_5d_lane(kdst + lane * p.bs * p.nkb * p.swb, &p.tmK, bar, 0, 0, 0, 0, l * p.fl + blk * p.fb + g);
      else
        for (int kb = 0; kb < p.nkb; ++kb)
          tma_load_5d_lane(kdst + kb * (kTileM * p.swb) + lane * p.bs * p.swb, &p.tmK, bar, kb * p.W, g, 0, blk, l);
    }
    __syncwarp();
  }
}

// The job's block-table entries -> SMEM (once per job, all lanes).
__device__ __noinline__ void paged_job_table(const FusedParams& p, const Job& jb, int lane, int* bts) {
  __syncwarp();
  if (jb.t_hi > jb.t_lo) {
    const long long b0 = (long long)jb.t_lo * kTileM / p.bs;
    const long long b1 = min(((long long)jb.t_hi * kTileM + p.bs - 1) / p.bs, (long long)p.max_blocks);
    const int* bt = p.btab + (long long)jb.b * p.max_blocks;
    for (long long i = b0 + lane; i < b1; i += 32) bts[i - b0] = bt[i];
  }
  __syncwarp();
}

// Row f3 producer (whole warp 0): the contiguous producer's loop with the K
// tiles read through the block table (out of line: the contiguous producer's
// code stays as it was -- the warp roles share the instruction cache).
__device__ __noinline__ void producer_paged(const FusedParams& p, uint8_t* smem, uint32_t bar_full, uint32_t bar_empty,
                                            uint32_t bar_qfull, uint32_t bar_qempty, int lane) {
  uint32_t stage = 0, sphase = 0, ui = 0;
  int* bts = reinterpret_cast<int*>(smem + p.off_bt);
  for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
    const Job jb = decode_job(p, job);
    paged_job_table(p, jb, lane, bts);
    for (int u = jb.u_lo; u < jb.u_hi; ++u, ++ui) {
      const int l = u / p.Hkv, g = u % p.Hkv;
      const uint32_t qs = ui & (p.nq - 1), qpar = (ui / p.nq) & 1;
      mbar_wait(bar_qempty + 8 * qs, qpar ^ 1);
      mbar_expect_tx(bar_qfull + 8 * qs, (uint32_t)(p.NC * p.d * p.esz));
      const uint32_t qdst = smem_u32(smem + p.off_q + qs * p.q_slot_bytes);
      for (int kb = 0; kb < p.nkb; ++kb)
        tma_load_5d(qdst + kb * (p.NCP * p.swb), &p.tmQ, bar_qfull + 8 * qs, kb * p.W, g * p.G, 0, l, jb.b);
      for (int t = jb.t_lo; t < jb.t_hi; ++t) {
        mbar_wait(bar_empty + 8 * stage, sphase ^ 1);
        const uint32_t kdst = smem_u32(smem + p.off_k + stage * p.k_stage_bytes);
        paged_tile(p, kdst, bar_full + 8 * stage, jb, t, g, l, lane, bts);
        if (++stage == (uint32_t)p.stages) { stage = 0; sphase ^= 1; }
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel
// Online (max, sum) merge in the log2 domain: (m, s) <- (m, s) (+) (m2, s2),
// s = sum 2^(x - m).  Empty partials are (-inf, 0); two empties stay empty.
__device__ __forceinline__ void merge2(float& m, float& s, float m2, float s2) {
  const float M = fmaxf(m, m2);
  const float Ms = (M == -CUDART_INF_F) ? 0.f : M;
  s = s * ex2(m - Ms) + s2 * ex2(m2 - Ms);
  m = M;
}

// Transposed butterfly merge of 32 columns x 32 lanes of (m, s) pairs: lane l
// returns column l merged over all 32 lanes.  31 merges per lane.
__device__ __forceinline__ void transpose_merge32(float (&m)[32], float (&s)[32], int lane, float& mo, float& so) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = lane & w;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float sm = up ? m[i] : m[i + w], ss = up ? s[i] : s[i + w];
      float km = up ? m[i + w] : m[i], ks = up ? s[i + w] : s[i];
      merge2(km, ks, __shfl_xor_sync(0xffffffffu, sm, w), __shfl_xor_sync(0xffffffffu, ss, w));
      m[i] = km;
      s[i] = ks;
    }
  }
  mo = m[0];
  so = s[0];
}

// Transposed butterfly sum of 32 columns x 32 lanes: lane l returns column l
// summed over all 32 lanes (fixed order, deterministic).  31 adds per lane.
__device__ __forceinline__ float transpose_add32(float (&s)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = lane & w;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? s[i] : s[i + w];
      const float keep = up ? s[i + w] : s[i];
      s[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return s[0];
}

// Bounded spin deadline: every in-kernel wait gives up (SP_ETIMEOUT) after
// kSpinNs of globaltimer, well before mbar_wait_slow's 4 s trap.
constexpr unsigned long long kSpinNs = 2000000000ull;

// Sequence-sharded peer exchange (world > 1), gather warp, one column, after
// the rank's n_tg CTA partials were merged into (M, S) (the single-GPU
// gather): the unit's designated CTA (token group u mod n_tg: spread evenly)
// stores that rank word into row `rank` of every peer's rank-word buffer
// (NVLink stores, this launch's parity half; the same row of the other half is
// re-zeroed for the launch after next); then the world rank words are merged
// in rank order -- the own one from registers, bit-identical to what the peers
// read -- so every rank computes the same lse2 bits.  The peers' words are
// polled together (one round trip).  Inline: the gather's code stays in one
// place: it runs inside peer_gather_unit.
__device__ __forceinline__ void peer_merge_col(const FusedParams& p, const unsigned long long* rw, bool designated,
                                               uint32_t parity, long long fin_half, int NCP, float& M, float& S) {
  const unsigned long long own = S > 0.f ? pack_ms(M, S) : pack_ms(-CUDART_INF_F, -1.f);   // never 0
  if (designated) {
    for (int r = 0; r < p.world; ++r) {
      if (r == p.rank) continue;
      unsigned long long* dst = p.peer[r] + (rw - p.peer[p.rank]) + (long long)p.rank * NCP;
      st_relaxed_sys_u64(dst + parity * fin_half, own);
      dst[(parity ^ 1u) * fin_half] = 0ull;
    }
  }
  const unsigned long long* cur = rw + parity * fin_half;
  unsigned long long v[kMaxPeers];
  unsigned missing = 0;
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r) {
    v[r] = (r < p.world && r != p.rank) ? ld_relaxed_sys_u64(cur + (long long)r * NCP) : own;
    missing |= (v[r] == 0ull ? 1u : 0u) << r;
  }
  unsigned long long t_dead = 0;
  for (long long it = 0; __any_sync(0xffffffffu, missing != 0); ++it) {
    __nanosleep(64);
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (missing & (1u << r)) {
        v[r] = ld_relaxed_sys_u64(cur + (long long)r * NCP);
        if (v[r] != 0ull) missing &= ~(1u << r);
      }
    if ((it & 1023) == 1023) {
      const unsigned long long now = globaltimer_ns();
      if (t_dead == 0) t_dead = now + kSpinNs;
      else if (now > t_dead) { set_err(p.err, kDevTimeout); missing = 0; }
    }
  }
  M = -CUDART_INF_F;
  S = 0.f;
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r) {
    if (r < p.world && v[r] != 0ull) {
      const float2 w = unpack_ms(v[r]);
      if (w.y > 0.f) merge2(M, S, w.x, w.y);
    }
  }
}

// Sequence-sharded gather of one unit (whole warp): the rank's n_tg partials
// (the single-GPU gather's loop), then peer_merge_col, then lse2 (+ the
// look-ahead keys' share, Z2') into ls.  Out of line, once per unit: the
// single-GPU gather's code stays exactly as it is (measured: inlining this
// path into the gather loop cost the single-GPU kernel 3 %).
__device__ __noinline__ void peer_gather_unit(const FusedParams& p, long long ubase, bool designated,
                                              const unsigned long long* part_cur, uint32_t parity, int NCP, int lane,
                                              float* ls) {
  const unsigned long long* src = part_cur + ubase * p.n_tg * NCP;
  const int ntg = p.n_tg;
  const long long fin_half = (long long)p.B * p.U * p.world * NCP;
  for (int c = lane; c < NCP; c += 32) {
    float M = -CUDART_INF_F, S = 0.f;
    for (int s0 = 0; s0 < ntg; s0 += kMaxLseBatch) {
      unsigned long long v[kMaxLseBatch];
      unsigned long long missing = 0;
#pragma unroll
      for (int j = 0; j < kMaxLseBatch; ++j) {
        v[j] = (s0 + j < ntg) ? ld_relaxed_sys_u64(src + (long long)(s0 + j) * NCP + c) : pack_ms(0.f, -1.f);
        missing |= (v[j] == 0ull ? 1ull : 0ull) << j;
      }
      long long it = 0;
      unsigned long long t_dead = 0;
      while (__any_sync(0xffffffffu, missing != 0)) {
        __nanosleep(it < 8 ? 64 : 200);
#pragma unroll
        for (int j = 0; j < kMaxLseBatch; ++j) {
          if (missing & (1ull << j)) {
            v[j] = ld_relaxed_sys_u64(src + (long long)(s0 + j) * NCP + c);
            if (v[j] != 0ull) missing &= ~(1ull << j);
          }
        }
        if ((++it & 1023) == 0 && t_dead == 0) t_dead = globaltimer_ns() + kSpinNs;
        if (t_dead != 0 && (it & 1023) == 0 && globaltimer_ns() > t_dead) {
          set_err(p.err, kDevTimeout);
#pragma unroll
          for (int j = 0; j < kMaxLseBatch; ++j)
            if (missing & (1ull << j)) v[j] = pack_ms(0.f, -1.f);
          missing = 0;
        }
      }
#pragma unroll
      for (int j = 0; j < kMaxLseBatch; ++j) {
        const float2 w = unpack_ms(v[j]);
        if (w.y > 0.f) merge2(M, S, w.x, w.y);
      }
    }
    peer_merge_col(p, p.peer[p.rank] + ubase * p.world * NCP + c, designated, parity, fin_half, NCP, M, S);
    if (p.la != nullptr && c < p.NC) {                           // the look-ahead keys' share (Z2')
      const float2 v = p.la[ubase * NCP + c];
      if (v.y > 0.f) merge2(M, S, v.x, v.y);
    }
    float l2 = 0.f;
    if (c < p.NC) {
      l2 = M + log2f(S);
      if (!isfinite(l2)) set_err(p.err, kDevNonFinite);
    }
    ls[c] = l2;
  }
}

// Debug timeline of the epilogue (-DSP_CHUNK_TRACE builds only): per CTA,
// [0] the job's last unit folded, [1] chunk phase entered, [2] neighbours ready,
// [3] chunk phase done (globaltimer).
#ifdef SP_CHUNK_TRACE
__device__ unsigned long long g_chunk_trace[160][8];
#define CHUNK_STAMP(k) \
  do { if ((threadIdx.x & 127) == 0) { g_chunk_trace[blockIdx.x % 160][k] = globaltimer_ns(); } } while (0)
#define CHUNK_STAMP0(k) \
  do { if (threadIdx.x == 0) { g_chunk_trace[blockIdx.x % 160][k] = globaltimer_ns(); } } while (0)
#else
#define CHUNK_STAMP(k) do { } while (0)
#define CHUNK_STAMP0(k) do { } while (0)
#endif

// Selection phase A in the score kernel's epilogue (sp_score_select; SURVEY
// 8(a) rows a7-a8: "1D average pooling", then "chunk the context contiguously
// and average").  Called by the CTA that completed a token group's
// importance.  A chunk whose pooling windows stay inside the token group is
// computed right here; the chunks whose windows cross the boundary with a
// neighbouring token group are computed by whichever of the two groups
// completes second (one self-resetting counter per boundary) -- nobody waits.
// Same arithmetic, same order as the selection kernel's phase A
// (select_body.cuh: centred window with shrinking edges, Z6; warp-tree sums for
// power-of-two chunks <= 32, else a rotated fixed order; mean over the chunk's
// true size, Z8), so the chunk scores -- and the selection -- are bit-identical
// to sp_select's.  128 threads (the aggregation warps), named barrier 2; sm: the
// acc region (free after the epilogue).  Out of line: once per job.
__device__ __noinline__ void chunk_phase(const FusedParams& p, const Job& jb, float* sm, int tok) {
  const long long n = jb.n, chunk = p.chunk, w = (p.pool_k - 1) / 2;
  const long long n_c = (n + chunk - 1) / chunk;
  const long long g_lo = (long long)jb.t_lo * kTileM, g_hi = min((long long)jb.t_hi * kTileM, n);
  const bool has_l = jb.tg > 0, has_r = jb.tg + 1 < p.n_tg;
  // chunks whose windows cross token boundary B: c*chunk - w < B <= (c+1)*chunk - 1 + w
  auto first_x = [&](long long B) { const long long v = B - w - chunk + 1; return v <= 0 ? 0LL : (v + chunk - 1) / chunk; };
  auto last_x = [&](long long B) { return min(n_c - 1, (B + w - 1) / chunk); };
  long long lo_c = (g_lo + chunk - 1) / chunk, hi_c = (g_hi + chunk - 1) / chunk;   // chunks starting here
  if (has_l) lo_c = max(lo_c, last_x(g_lo) + 1);
  if (has_r) hi_c = min(hi_c, first_x(g_hi));
  volatile int* flag = reinterpret_cast<volatile int*>(sm);
  CHUNK_STAMP(1);
  if (tok == 0) {
    __threadfence();                                   // this token group's importance before the counts
    unsigned* bc = p.bnd_cnt + (long long)jb.b * p.n_tg;
    const unsigned ol = has_l ? atomicAdd(bc + jb.tg - 1, 1u) : 0u;   // boundary (tg-1 | tg)
    const unsigned orr = has_r ? atomicAdd(bc + jb.tg, 1u) : 0u;      // boundary (tg | tg+1)
    const bool dl = has_l && ol == 1u, dr = has_r && orr == 1u;
    if (dl) bc[jb.tg - 1] = 0u;                        // second arrival: reset for the next launch
    if (dr) bc[jb.tg] = 0u;
    if (dl || dr) __threadfence();                     // the neighbour's importance
    flag[0] = dl ? 1 : 0;
    flag[1] = dr ? 1 : 0;
  }
  named_bar(2, 128);
  const bool dl = flag[0] != 0, dr = flag[1] != 0;
  named_bar(2, 128);
  CHUNK_STAMP(2);
  if (dl) lo_c = first_x(g_lo);
  if (dr) hi_c = last_x(g_hi) + 1;
  if (lo_c >= hi_c) return;
  const long long a0 = lo_c * chunk, a1 = min(hi_c * chunk, n);     // pooled tokens
  const long long lo = max(0LL, a0 - w), hi = min(n, a1 + w);        // staged importance
  const int ns = (int)(hi - lo), np = (int)(a1 - a0);
  float* sb = sm;                                                   // [ns] importance
  float* pb = sm + ((ns + 3) & ~3);                                 // [np] pooled
  const float* imp = p.imp + (long long)jb.b * p.N + lo;
  for (int j0 = 0; j0 < ns; j0 += 16 * kTileM) {                    // all loads of a batch in flight
    float r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int j = j0 + k * kTileM + tok;
      r[k] = j < ns ? __ldcg(imp + j) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int j = j0 + k * kTileM + tok;
      if (j < ns) sb[j] = r[k];
    }
  }
  named_bar(2, 128);
  const float inv_k = 1.f / (float)p.pool_k;
  for (int i = tok; i < np; i += kTileM) {
    const long long t = a0 + i;
    float ws = 0.f;
    if (t >= w && t + w <= n - 1) {                                 // interior: full window
      const float* q = sb + (t - w - lo);
      for (int k = 0; k < p.pool_k; ++k) ws += q[k];
      pb[i] = ws * inv_k;
    } else {                                                        // sequence edges: shrink
      const long long e0 = t - w < 0 ? 0 : t - w, e1 = t + w > n - 1 ? n - 1 : t + w;
      for (long long j = e0; j <= e1; ++j) ws += sb[j - lo];
      pb[i] = ws / (float)(e1 - e0 + 1);
    }
  }
  named_bar(2, 128);
  float* cs = p.cs_out + (long long)jb.b * p.n_c_row;
  if (chunk <= 32 && (chunk & (chunk - 1)) == 0) {
    const int lg = __ffs((int)chunk) - 1, lane = tok & 31;
    for (int g0 = (tok >> 5) * 32; g0 < np; g0 += kTileM) {         // 32-token windows on chunk boundaries
      float v = g0 + lane < np ? pb[g0 + lane] : 0.f;
      for (int o = (int)chunk >> 1; o >= 1; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, (int)chunk);
      if ((lane & ((int)chunk - 1)) == 0 && g0 + lane < np) {
        const long long c = lo_c + ((g0 + lane) >> lg);
        cs[c] = v / (float)(min((c + 1) * chunk, n) - c * chunk);
      }
    }
  } else {
    for (long long c = lo_c + tok; c < hi_c; c += kTileM) {
      const long long t0 = c * chunk, t1 = min((c + 1) * chunk, n);
      const int m = (int)(t1 - t0), ii = (int)(t0 - a0), rot = (int)(c % m);
      float sacc = 0.f;
      for (int j = 0; j < m; ++j) {
        int k = j + rot;
        if (k >= m) k -= m;
        sacc += pb[ii + k];
      }
      cs[c] = sacc / (float)m;
    }
  }
  CHUNK_STAMP(3);
}

// kG: compile-time GQA group size (1, 2, 4, 8) or 0 for any G.  One
// instantiation per group size keeps the kernel's hot code small: the warp
// roles run different code concurrently on each SMSP and share the
// instruction cache.
// kF8: e4m3 inputs (row f4), kind::f8f6f4 MMA; everything after the MMA is shared.
template <int kG, int kNCP, bool kF8>
__global__ void __launch_bounds__(kThreads, 1) k_fused(const __grid_constant__ FusedParams p) {
  // kNCP > 0: compile-time padded column count (one 32-column TMEM group for
  // the 8B geometry): the per-tile loops become straight-line code
  const int NCP = kNCP > 0 ? kNCP : p.NCP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base as an offset into the __shared__ array, so the
  // compiler keeps the address space: LDS/STS/ATOMS instead of generic accesses
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // warp index broadcast from lane 0: provably warp-uniform, so each role's
  // loop state (descriptors, coordinates, phases) lives in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  // barrier map: full[S] empty[S] qfull[kMaxQSlots] qempty[kMaxQSlots] tfull[kMaxSlots] tempty[kMaxSlots]
  //              rfull[2] rempty[2] lfull[kLseRing] lempty[kLseRing]; then the TMEM base address
  const uint32_t bar_full = smem_u32(bars), bar_empty = bar_full + 8 * p.stages;
  const uint32_t bar_qfull = bar_empty + 8 * p.stages, bar_qempty = bar_qfull + 8 * kMaxQSlots;
  const uint32_t bar_tfull = bar_qempty + 8 * kMaxQSlots, bar_tempty = bar_tfull + 8 * kMaxSlots;
  const uint32_t bar_rfull = bar_tempty + 8 * kMaxSlots, bar_rempty = bar_rfull + 16;
  const uint32_t bar_lfull = bar_rempty + 16, bar_lempty = bar_lfull + 8 * kLseRing;
  uint32_t* tmem_base_s =
      reinterpret_cast<uint32_t*>(bars + 2 * p.stages + 2 * kMaxQSlots + 2 * kMaxSlots + 4 + 2 * kLseRing);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(bar_tfull + 8 * s, 1);
      mbar_init(bar_tempty + 8 * s, 4);
    }
    for (int s = 0; s < kMaxQSlots; ++s) {
      mbar_init(bar_qfull + 8 * s, 1);
      mbar_init(bar_qempty + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_rfull + 8 * s, 128);
      mbar_init(bar_rempty + 8 * s, 1);
    }
    for (int s = 0; s < kLseRing; ++s) {
      mbar_init(bar_lfull + 8 * s, 32);
      mbar_init(bar_lempty + 8 * s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&p.tmK);
    prefetch_tmap(&p.tmQ);
  }
  // zero both Q slots once: rows >= NC (MMA padding columns) are never written by TMA
  for (uint32_t o = threadIdx.x * 16; o < (uint32_t)p.nq * p.q_slot_bytes; o += kThreads * 16)
    *reinterpret_cast<uint4*>(smem + p.off_q + o) = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_s)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // every CTA is resident (cooperative launch): a programmatic dependent (the
  // selection) may be scheduled now and waits for this grid in griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t tmem = *tmem_base_s;
  const uint32_t nslots = (uint32_t)p.nslots;
  // this launch publishes into part[parity]; part[parity ^ 1] (the previous
  // launch's) is re-zeroed off the critical path, for the launch after next
  const uint32_t parity = ld_acquire(p.epoch) & 1u;
  const long long part_half = (long long)p.B * p.U * p.n_tg * NCP;
  unsigned long long* const part_cur = p.part + parity * part_half;
  unsigned long long* const part_old = p.part + (parity ^ 1u) * part_half;

  if (warp == 0 && p.paged) {
    // ================================================================ TMA producer, paged K (row f3)
    producer_paged(p, smem, bar_full, bar_empty, bar_qfull, bar_qempty, lane);
  } else if (warp == 0) {
    // ================================================================ TMA producer
    // (whole warp, warp-uniform loop; the helpers issue from one elected lane)
    {
      uint32_t stage = 0, sphase = 0, ui = 0;
      unsigned long long w_empty = 0, w_q = 0;
      uint64_t l2pol = 0;
      if (p.l2hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(l2pol));
      for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
        const Job jb = decode_job(p, job);
        for (int u = jb.u_lo; u < jb.u_hi; ++u, ++ui) {
          const int l = u / p.Hkv, g = u % p.Hkv;
          const uint32_t qs = ui & (p.nq - 1), qpar = (ui / p.nq) & 1;
          mbar_wait_acc(p, bar_qempty + 8 * qs, qpar ^ 1, w_q);
          trace_stamp(p, ui, 0);
          mbar_expect_tx(bar_qfull + 8 * qs, (uint32_t)(p.NC * p.d * p.esz));
          const uint32_t qdst = smem_u32(smem + p.off_q + qs * p.q_slot_bytes);
          #pragma unroll 1
          for (int kb = 0; kb < p.nkb; ++kb)
            tma_load_5d(qdst + kb * (NCP * p.swb), &p.tmQ, bar_qfull + 8 * qs, kb * p.W, g * p.G, 0, l, jb.b);
          for (int t = jb.t_lo; t < jb.t_hi; ++t) {
            mbar_wait_acc(p, bar_empty + 8 * stage, sphase ^ 1, w_empty);
            mbar_expect_tx(bar_full + 8 * stage, p.k_stage_bytes);
            const uint32_t kdst = smem_u32(smem + p.off_k + stage * p.k_stage_bytes);
            if (p.l2hint) {
              #pragma unroll 1
              for (int kb = 0; kb < p.nkb; ++kb)
                tma_load_5d_hint(kdst + kb * (kTileM * p.swb), &p.tmK, bar_full + 8 * stage, kb * p.W, t * kTileM, g,
                                 l, jb.b, l2pol);
            } else {
              #pragma unroll 1
              for (int kb = 0; kb < p.nkb; ++kb)
                tma_load_5d(kdst + kb * (kTileM * p.swb), &p.tmK, bar_full + 8 * stage, kb * p.W, t * kTileM, g, l,
                            jb.b);
            }
            if (++stage == (uint32_t)p.stages) { stage = 0; sphase ^= 1; }
          }
        }
      }
      trace_waits(p, 0, w_empty);
      trace_waits(p, 1, w_q);
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    // Each tile's logits D[128 x NCP] go to the next slot of a ring of nslots
    // TMEM tile slots; a slot is released by the aggregation warps once they
    // have folded that tile (tile-granular reuse hides the exchange latency).
    // Whole warp, warp-uniform loop; umma_* issue from one elected lane.
    {
      uint32_t stage = 0, sphase = 0, ui = 0, gt = 0, gslot = 0, gph = 0;
      unsigned long long w_qf = 0, w_slot = 0, w_full = 0, w_issue = 0;
      const long long t_start = kTrace ? clock64() : 0;
      // UMMA smem descriptors: the high word (SBO, version, swizzle) is constant;
      // the low word is (address >> 4) | LBO and a K step just adds to it.
      const uint32_t desc_hi = (uint32_t)(make_sdesc(0, 8 * p.swb, p.layout_type) >> 32);
      // kb-interleaved K tiles (paged, one box per block): 8-row groups of all kb
      // halves adjacent, so the A operand's group stride is nkb * 1024 B and its
      // kb step 1024 B (generic issue loop); otherwise the straight-line paths
      const uint32_t a_hi = p.kinter ? (uint32_t)(make_sdesc(0, 8 * p.swb * p.nkb, p.layout_type) >> 32) : desc_hi;
      const uint32_t a_kb = (p.kinter ? 8 * p.swb : kTileM * p.swb) >> 4, b_kb = (NCP * p.swb) >> 4;
      const int ksteps = p.ksteps;
      // (measured: kb-interleaved tiles run faster through the generic loop than
      // through a straight-line sequence, 0.41 vs 0.46 ms at C3 block size 16)
      const int fast = p.kinter || ksteps != 4 ? 0 : p.nkb;
      for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
        const Job jb = decode_job(p, job);
        for (int u = jb.u_lo; u < jb.u_hi; ++u, ++ui) {
          const uint32_t qs = ui & (p.nq - 1), qpar = (ui / p.nq) & 1;
          mbar_wait_acc(p, bar_qfull + 8 * qs, qpar, w_qf);
          const uint32_t b_lo0 = ((smem_u32(smem + p.off_q + qs * p.q_slot_bytes) >> 4) & 0x3FFFu) | (1u << 16);
          for (int t = jb.t_lo; t < jb.t_hi; ++t, ++gt) {
            const uint32_t slot = gslot;
            unsigned long long* tt = (kTrace && p.tile_trace != nullptr && blockIdx.x == 0 && gt < 1000)
                                         ? p.tile_trace + gt * 8 : nullptr;
            if (tt && lane == 0) { tt[0] = clock64(); tt[4] = globaltimer_ns(); }
            mbar_wait_acc(p, bar_tempty + 8 * slot, gph ^ 1, w_slot);
            if (tt && lane == 0) tt[1] = clock64();
            if (++gslot == nslots) { gslot = 0; gph ^= 1; }
            if (t == jb.t_lo) trace_stamp(p, ui, 1);
            mbar_wait_acc(p, bar_full + 8 * stage, sphase, w_full);
            if (tt && lane == 0) tt[2] = clock64();
            tc_fence_after();
            const uint32_t a_lo0 = ((smem_u32(smem + p.off_k + stage * p.k_stage_bytes) >> 4) & 0x3FFFu) | (1u << 16);
            const uint32_t dcol = tmem + slot * NCP;
            const long long ti0 = kTrace ? clock64() : 0;
            // straight-line issue for the common head dims (d = 64, 128, 256 with
            // 64-element swizzle blocks): the descriptor arithmetic pipelines
            // across the MMAs (a loop back-edge halves the issue rate)
            if (fast == 2) {
              issue_tile<8, 4, kF8>(dcol, a_lo0, b_lo0, desc_hi, b_kb, p.idesc);
            } else if (fast == 1) {
              issue_tile<4, 4, kF8>(dcol, a_lo0, b_lo0, desc_hi, b_kb, p.idesc);
            } else if (fast == 4) {
              issue_tile<16, 4, kF8>(dcol, a_lo0, b_lo0, desc_hi, b_kb, p.idesc);
            } else {
              uint32_t accum = 0;
#pragma unroll 1
              for (int kb = 0; kb < p.nkb; ++kb) {
                uint32_t a_lo = a_lo0 + kb * a_kb, b_lo = b_lo0 + kb * b_kb;
#pragma unroll 1
                for (int ks = 0; ks < ksteps; ++ks, a_lo += 2, b_lo += 2) {
                  umma<kF8>(dcol, ((uint64_t)a_hi << 32) | a_lo, ((uint64_t)desc_hi << 32) | b_lo, p.idesc, accum);
                  accum = 1;
                }
              }
            }
            umma_commit(bar_empty + 8 * stage);
            umma_commit(bar_tfull + 8 * slot);
            if (kTrace && p.trace != nullptr) w_issue += clock64() - ti0;
            if (tt && lane == 0) { tt[3] = clock64(); tt[5] = globaltimer_ns(); }
            if (++stage == (uint32_t)p.stages) { stage = 0; sphase ^= 1; }
          }
          umma_commit(bar_qempty + 8 * qs);
        }
      }
      trace_waits(p, 2, w_qf);
      trace_waits(p, 3, w_slot);
      trace_waits(p, 4, w_full);
      trace_waits(p, 5, kTrace ? clock64() - t_start : 0);
      trace_waits(p, 6, w_issue);
    }
  } else if (warp >= kStatsWarp0 && warp < kFinalWarp0 && p.mode != kModeFinish) {
    // ================================================================ softmax statistics
    // Progressive: each tile is folded as soon as its MMA completes into a
    // per-thread running sum 2^(x*xs - ref) per column.  The reference is
    // shared by the warp: lane 0's value in the unit's first tile (a lane whose
    // value later exceeds it by > 2^64 re-bases its own reference -- rare --
    // which keeps fp32 finite).  One exp2 per logit, no per-tile shuffles; at
    // the end of the unit a transposed butterfly sum gives the warp's (ref,
    // sum) per column (a full (max, sum) merge only if some lane re-based).
    // The exchange warp merges the 4 warps and publishes.
    const int q = warp & 3;                       // TMEM lane quarter
    float2* red = reinterpret_cast<float2*>(smem + p.off_red);   // [2][4][NCP]
    uint32_t ui = 0, gt = 0;
    for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
      const Job jb = decode_job(p, job);
      const long long tok0 = (long long)jb.t_lo * kTileM + q * 32 + lane;
      for (int u = jb.u_lo; u < jb.u_hi; ++u, ++ui) {
        const uint32_t gt0 = gt;
        uint32_t slot0 = gt % nslots, ph0 = (gt / nslots) & 1;
        float2* rb = red + (ui & 1) * 4 * NCP;
        mbar_wait(bar_rempty + 8 * (ui & 1), ((ui >> 1) & 1) ^ 1);   // exchange warp done with rb
        if (q == 0 && lane == 0) trace_stamp(p, ui, 2);
#pragma unroll 1
        for (int grp = 0; grp < NCP / 32; ++grp) {
          float ref[32], sum[32];
          float myref = 0.f;                                            // ref of column 32*grp + lane
          bool rebased = false;
          gt = gt0;
          uint32_t slot = slot0, ph = ph0;
          for (int t = jb.t_lo; t < jb.t_hi; ++t, ++gt) {
            mbar_wait(bar_tfull + 8 * slot, ph);
            tc_fence_after();
            float x[32];
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + slot * NCP + grp * 32;
            float* x0 = x;
            tmem_ld16_issue(ta, *reinterpret_cast<float(*)[16]>(x0));
            tmem_ld16_issue(ta + 16, *reinterpret_cast<float(*)[16]>(x0 + 16));
            tmem_wait();
            tie16(*reinterpret_cast<float(*)[16]>(x0));
            tie16(*reinterpret_cast<float(*)[16]>(x0 + 16));
            if (t == jb.t_lo) {
              // lane 0's token is valid whenever any lane's is (lowest index)
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                ref[i] = __shfl_sync(0xffffffffu, x[i] * p.xs, 0);
                myref = lane == i ? ref[i] : myref;
                sum[i] = 0.f;
              }
            }
            if (tok0 + (long long)(t - jb.t_lo) * kTileM < jb.n) {
              {
                // d = y - ref; the common case adds 2^d (FFMA, MUFU, FADD + a max);
                // a jump d > 64 (rare) re-bases that column on y to keep fp32 finite
                float dmax = -CUDART_INF_F;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  x[i] = fmaf(x[i], p.xs, -ref[i]);
                  dmax = fmaxf(dmax, x[i]);
                }
                if (dmax <= 64.f) {
#pragma unroll
                  for (int i = 0; i < 32; ++i) sum[i] += ex2(x[i]);
                } else {
                  rebased = true;
#pragma unroll
                  for (int i = 0; i < 32; ++i) {
                    const bool big = x[i] > 64.f;
                    const float e = ex2(big ? -x[i] : x[i]);
                    sum[i] = big ? fmaf(sum[i], e, 1.f) : sum[i] + e;
                    ref[i] = big ? ref[i] + x[i] : ref[i];
                  }
                }
              }
            }
            if (p.mode == kModeStats && grp + 1 == NCP / 32) {
              // statistics-only launch: no aggregation reads the tile, release it here
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(bar_tempty + 8 * slot);
            }
            if (++slot == nslots) { slot = 0; ph ^= 1; }
          }
          float mo, so;
          if (__any_sync(0xffffffffu, rebased)) {
            transpose_merge32(ref, sum, lane, mo, so);                  // references differ (rare)
          } else {
            so = transpose_add32(sum, lane);                            // column 32*grp + lane
            mo = myref;
          }
          rb[q * NCP + grp * 32 + lane] = make_float2(mo, so);
        }
        if (q == 0 && lane == 0) trace_stamp(p, ui, 7);
        mbar_arrive(bar_rfull + 8 * (ui & 1));                        // 128 arrivals: all columns written
      }
    }
  } else if (warp == 2 && p.mode != kModeFinish) {
    // ================================================================ statistics exchange
    // Merge the 4 statistics warps into the CTA partial and publish it: one
    // 64-bit word (max2, sum) per column, single-copy atomic, so a reader sees
    // either 0 (not yet written) or the complete pair -- no flag, no fence.
    const float2* red = reinterpret_cast<const float2*>(smem + p.off_red);   // [2][4][NCP]
    uint32_t ui = 0;
    for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
      const Job jb = decode_job(p, job);
      for (int u = jb.u_lo; u < jb.u_hi; ++u, ++ui) {
        const long long ubase = (long long)jb.b * p.U + u;
        mbar_wait(bar_rfull + 8 * (ui & 1), (ui >> 1) & 1);
        const float2* rb = red + (ui & 1) * 4 * NCP;
        const long long row = (ubase * p.n_tg + jb.tg) * NCP;
        for (int c = lane; c < NCP; c += 32) {
          float mm = -CUDART_INF_F, ss = 0.f;
          if (c < p.NC) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {                                // a warp with no valid token has sum 0
              const float2 v = rb[w * NCP + c];                           // and an undefined ref: merge it as -inf
              merge2(mm, ss, v.y > 0.f ? v.x : -CUDART_INF_F, v.y);
            }
          }
          if (!(ss > 0.f) || jb.t_lo == jb.t_hi) { mm = -CUDART_INF_F; ss = -1.f; }   // written, but empty
                                                                        // (an empty job of a ragged batch)
          st_relaxed_u64(part_cur + row + c, pack_ms(mm, ss));
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(bar_rempty + 8 * (ui & 1));
          trace_stamp(p, ui, 3);
        }
      }
    }
    // re-zero this CTA's rows of the previous launch's buffer (read by nobody now)
    for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
      const Job jb = decode_job(p, job);
      for (int u = jb.u_lo; u < jb.u_hi; ++u) {
        const long long row = (((long long)jb.b * p.U + u) * p.n_tg + jb.tg) * NCP;
        for (int c = lane; c < NCP; c += 32) part_old[row + c] = 0ull;
      }
      if (jb.ug == 0 && lane == 0)                                  // the token group's counter of the previous
        p.fin_cnt[((long long)(parity ^ 1u) * p.B + jb.b) * p.n_tg + jb.tg] = 0u;   // launch parity
    }
  } else if (warp == 3 && p.mode != kModeStats) {
    // ================================================================ lse2 gather
    // Polls the unit's n_tg published partials (all loads of a batch in flight
    // together; zero words are re-read until written), merges them in
    // token-group order -- every CTA computes the same lse2 bit for bit -- and
    // stages lse2 in SMEM for the aggregation warps.
    float* lse_s = reinterpret_cast<float*>(smem + p.off_lse);    // [kLseRing][NCP]
    uint32_t ui = 0;
    for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
      const Job jb = decode_job(p, job);
      for (int u = jb.u_lo; u < jb.u_hi; ++u, ++ui) {
        const uint32_t par = ui % kLseRing;
        const long long ubase = (long long)jb.b * p.U + u;
        mbar_wait(bar_lempty + 8 * par, ((ui / kLseRing) & 1) ^ 1);    // aggregation done with ls[par]
        float* ls = lse_s + par * NCP;
        const unsigned long long* src = part_cur + ubase * p.n_tg * NCP;
        const int ntg = p.n_tg;
        for (int c = lane; c < NCP && p.mode == kModeFinish; c += 32) {
          // lse2 supplied by the caller (sequence-sharded split: globally combined statistics)
          float l2 = 0.f;
          if (c < p.NC) {
            const int l = u / p.Hkv, g = u % p.Hkv;
            l2 = p.lse_in[(((long long)jb.b * p.L + l) * p.Hkv * p.G + g * p.G + c % p.G) * p.Rv + c / p.G];
          }
          ls[c] = l2;
        }
        if (p.world > 1 && p.mode == kModeFull)                        // sequence-sharded over GPUs
          peer_gather_unit(p, ubase, (u % p.n_tg) == jb.tg, part_cur, parity, NCP, lane, ls);
        for (int c = lane; c < NCP && p.mode == kModeFull && p.world == 1; c += 32) {
          float M = -CUDART_INF_F, S = 0.f;
          for (int s0 = 0; s0 < ntg; s0 += kMaxLseBatch) {
            unsigned long long v[kMaxLseBatch];
            unsigned long long missing = 0;
#pragma unroll
            for (int j = 0; j < kMaxLseBatch; ++j) {
              v[j] = (s0 + j < ntg) ? ld_relaxed_sys_u64(src + (long long)(s0 + j) * NCP + c) : pack_ms(0.f, -1.f);
              missing |= (v[j] == 0ull ? 1ull : 0ull) << j;
            }
            long long it = 0;
            unsigned long long t_dead = 0;
            while (__any_sync(0xffffffffu, missing != 0)) {
              __nanosleep(it < 8 ? 64 : 200);
#pragma unroll
              for (int j = 0; j < kMaxLseBatch; ++j) {
                if (missing & (1ull << j)) {
                  v[j] = ld_relaxed_sys_u64(src + (long long)(s0 + j) * NCP + c);
                  if (v[j] != 0ull) missing &= ~(1ull << j);
                }
              }
              if ((++it & 1023) == 0 && t_dead == 0) t_dead = globaltimer_ns() + kSpinNs;
              if (t_dead != 0 && (it & 1023) == 0 && globaltimer_ns() > t_dead) {
                set_err(p.err, kDevTimeout);
#pragma unroll
                for (int j = 0; j < kMaxLseBatch; ++j)
                  if (missing & (1ull << j)) v[j] = pack_ms(0.f, -1.f);
                missing = 0;
              }
            }
#pragma unroll
            for (int j = 0; j < kMaxLseBatch; ++j) {
              const float2 w = unpack_ms(v[j]);
              if (w.y > 0.f) merge2(M, S, w.x, w.y);
            }
          }
          if (p.la != nullptr && c < p.NC) {                         // the look-ahead keys' share (Z2')
            const float2 v = p.la[ubase * NCP + c];
            if (v.y > 0.f) merge2(M, S, v.x, v.y);
          }
          float l2 = 0.f;
          if (c < p.NC) {
            l2 = M + log2f(S);
            if (!isfinite(l2)) set_err(p.err, kDevNonFinite);
          }
          ls[c] = l2;
        }
        if (lane == 0) trace_stamp(p, ui, 5);
        mbar_arrive(bar_lfull + 8 * par);
        if (lane == 0) trace_stamp(p, ui, 4);
      }
    }
  } else if (warp >= kFinalWarp0 && p.mode != kModeStats) {
    // ================================================================ (l,h)-max aggregation
    const int q = warp & 3;
    float* acc = reinterpret_cast<float*>(smem + p.off_acc);      // [tpc][Rv][128]
    const float* lse_s = reinterpret_cast<const float*>(smem + p.off_lse);    // [kLseRing][NCP]
    const int tok = q * 32 + lane;
    uint32_t ui = 0, gt = 0;
    for (long long job = blockIdx.x; job < p.total_jobs; job += gridDim.x) {
      const Job jb = decode_job(p, job);
      const int ntile = jb.t_hi - jb.t_lo;
      for (int t = 0; t < ntile; ++t)
        for (int r = 0; r < p.Rv; ++r) acc[(t * p.Rv + r) * kTileM + tok] = -CUDART_INF_F;
      for (int u = jb.u_lo; u < jb.u_hi; ++u, ++ui) {
        const uint32_t par = ui % kLseRing;
        mbar_wait(bar_lfull + 8 * par, (ui / kLseRing) & 1);
        const float* ls = lse_s + par * NCP;
        uint32_t slot = gt % nslots, ph = (gt / nslots) & 1;
        if constexpr (kNCP == 32) {
          // one 32-column group: the unit's lse2 stays in registers for all its tiles
          float lv[32];
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            const float4 v4 = *reinterpret_cast<const float4*>(ls + 4 * i4);
            lv[4 * i4] = v4.x; lv[4 * i4 + 1] = v4.y; lv[4 * i4 + 2] = v4.z; lv[4 * i4 + 3] = v4.w;
          }
          for (int t = 0; t < ntile; ++t, ++gt) {
            mbar_wait(bar_tfull + 8 * slot, ph);
            tc_fence_after();
            {
              const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + slot * 32;
              float* arow = acc + (t * p.Rv) * kTileM + tok;
              float xa[16], xb[16];
              tmem_ld16_issue(ta, xa);
              tmem_ld16_issue(ta + 16, xb);
              tmem_wait();
              tie16(xa);
              tie16(xb);
              fold_tile<kG, 16>(xa, *reinterpret_cast<const float(*)[16]>(&lv[0]), p.xs, 0, p.NC, p.G, p.Rv, arow);
              fold_tile<kG, 16>(xb, *reinterpret_cast<const float(*)[16]>(&lv[16]), p.xs, 1, p.NC, p.G, p.Rv, arow);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_tempty + 8 * slot);         // release the TMEM tile slot
            if (++slot == nslots) { slot = 0; ph ^= 1; }
          }
        } else
        for (int t = 0; t < ntile; ++t, ++gt) {
          mbar_wait(bar_tfull + 8 * slot, ph);
          tc_fence_after();
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + slot * NCP;
          float* arow = acc + (t * p.Rv) * kTileM + tok;
#pragma unroll 1
          for (int k0 = 0; k0 < NCP / 16; k0 += 2) {
            float xa[16], xb[16];
            const bool two = k0 + 1 < NCP / 16;
            tmem_ld16_issue(ta + k0 * 16, xa);
            if (two) tmem_ld16_issue(ta + k0 * 16 + 16, xb);
            tmem_wait();
            tie16(xa);
            tie16(xb);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h == 1 && !two) break;
              const int k = k0 + h;
              float lv[16];
#pragma unroll
              for (int i4 = 0; i4 < 4; ++i4) {
                const float4 v4 = *reinterpret_cast<const float4*>(ls + k * 16 + 4 * i4);
                lv[4 * i4] = v4.x; lv[4 * i4 + 1] = v4.y; lv[4 * i4 + 2] = v4.z; lv[4 * i4 + 3] = v4.w;
              }
              fold_tile<kG, 16>(h == 0 ? xa : xb, lv, p.xs, k, p.NC, p.G, p.Rv, arow);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_tempty + 8 * slot);           // release the TMEM tile slot
          if (++slot == nslots) { slot = 0; ph ^= 1; }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_lempty + 8 * par);
        if (q == 0 && lane == 0) trace_stamp(p, ui, 6);
      }
      CHUNK_STAMP(0);
      // ---- job epilogue: importance = mean_r 2^acc (possibly across unit groups)
      //      or, head-sharded (acc_out), the log2-domain max itself for a max-reduce across ranks
      const float inv = 1.f / (float)p.Rv;
      if (p.n_ug == 1) {
        for (int t = 0; t < ntile; ++t) {
          const long long i = (long long)(jb.t_lo + t) * kTileM + tok;
          if (i < jb.n) {
            if (p.acc_out != nullptr) {
              for (int r = 0; r < p.Rv; ++r)
                p.acc_out[((long long)jb.b * p.Rv + r) * p.N + i] = acc[(t * p.Rv + r) * kTileM + tok];
              continue;
            }
            float s = 0.f;
            for (int r = 0; r < p.Rv; ++r) s += ex2(acc[(t * p.Rv + r) * kTileM + tok]);
            p.imp[(long long)jb.b * p.N + i] = s * inv;
          }
        }
        if (p.cs_out != nullptr) {                                  // selection phase A (sp_score_select)
          named_bar(2, 128);
          chunk_phase(p, jb, acc, tok);
          named_bar(2, 128);                                        // acc is the next job's
        }
      } else {
        for (int t = 0; t < ntile; ++t) {
          const long long i = (long long)(jb.t_lo + t) * kTileM + tok;
          if (i < jb.n)
            for (int r = 0; r < p.Rv; ++r)
              p.accpart[(((long long)jb.b * p.n_ug + jb.ug) * p.Rv + r) * p.acc_pitch + i] = acc[(t * p.Rv + r) * kTileM + tok];
        }
        if (p.defer) continue;                                      // the selection finalizes (sp_score_select)
        named_bar(2, 128);                                          // the CTA's partial maps, then one
        unsigned* fc = p.fin_cnt + ((long long)(p.mode == kModeFinish ? 2u : parity) * p.B + jb.b) * p.n_tg + jb.tg;
        if (threadIdx.x == kFinalWarp0 * 32) {
          __threadfence();
          atomicAdd(fc, 1u);
          spin_geq(fc, (unsigned)p.n_ug, p.err);
          __threadfence();
        }
        named_bar(2, 128);
        CHUNK_STAMP(4);
        // this CTA finalises slice ug of the token group's tokens: the max over
        // the n_ug unit groups' partial maps.  Every (group, row, token) value of
        // the slice is loaded with 16 loads in flight per thread (coalesced over
        // tokens) and folded into SMEM (red.shared: the generic atomic the
        // compiler emits for this pointer costs several microseconds here) with an order-preserving unsigned max
        // (order-free: the same bits as a sequential max); then mean_r 2^max in
        // row order.  (A per-token loop over the groups was a chain of dependent
        // L2 round trips: ~0.9 us per unit group at the end of every launch; fire-
        // and-forget global atomic maxima instead of the partial maps measured no
        // faster -- the L2 atomic rate.)
        const long long g_lo = (long long)jb.t_lo * kTileM;
        const long long g_hi = min((long long)jb.t_hi * kTileM, (long long)jb.n);
        const long long n = max(0LL, g_hi - g_lo);
        const long long s_lo = g_lo + n * jb.ug / p.n_ug, s_hi = g_lo + n * (jb.ug + 1) / p.n_ug;
        const int S = (int)(s_hi - s_lo), RS = p.Rv * S;
        unsigned* mx = reinterpret_cast<unsigned*>(acc);          // [Rv][S] (acc was copied out above)
        for (int e = tok; e < RS; e += kTileM) mx[e] = 0u;        // below every ordered key
        named_bar(2, 128);
        if (S > 0) {
          const float* src = p.accpart + (long long)jb.b * p.n_ug * p.Rv * p.acc_pitch + s_lo;
          const int tot = p.n_ug * RS;
          // element e = q*S + i (q = group*Rv + row), e = tok + k*128: the indices
          // advance by a fixed (dq, di) per step (no per-element division)
          const int dq = kTileM / S, di = kTileM - dq * S, dr = dq % p.Rv;
          int q = tok / S, i = tok - q * S, r = q % p.Rv;
          const long long pitch = p.acc_pitch, step = (long long)dq * pitch + di, wrap = pitch - S;
          const float* ptr = src + (long long)q * pitch + i;
#ifndef SP_EPI_KU
#define SP_EPI_KU 24
#endif
          constexpr int kU = SP_EPI_KU;                             // loads in flight per thread (32: 163 registers)
          for (int e0 = tok; e0 < tot; e0 += kU * kTileM) {
            float v[kU];
            int dst[kU];
#pragma unroll
            for (int k = 0; k < kU; ++k) {
              const bool in = e0 + k * kTileM < tot;
              dst[k] = in ? r * S + i : -1;
              v[k] = __ldcg(in ? ptr : src);                        // (branch-free: src is a valid address)
              i += di;
              r += dr;
              ptr += step;
              if (i >= S) { i -= S; ++r; ptr += wrap; }
              if (r >= p.Rv) r -= p.Rv;
            }
#pragma unroll
            for (int k = 0; k < kU; ++k) {
              if (dst[k] >= 0) {
                const unsigned u = __float_as_uint(v[k]);
                red_smem_max(smem_u32(&mx[dst[k]]), (u & 0x80000000u) ? ~u : (u | 0x80000000u));
              }
            }
          }
        }
        named_bar(2, 128);
        for (int i = tok; i < S; i += kTileM) {
          float s = 0.f;
          for (int r = 0; r < p.Rv; ++r) {
            const unsigned k = mx[r * S + i];
            const float m = __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
            if (p.acc_out != nullptr) p.acc_out[((long long)jb.b * p.Rv + r) * p.N + s_lo + i] = m;
            s += ex2(m);
          }
          if (p.acc_out == nullptr) p.imp[(long long)jb.b * p.N + s_lo + i] = s * inv;
        }
        named_bar(2, 128);
        CHUNK_STAMP(5);
        // a second count only where needed: finish mode resets its counter (the
        // full and statistics modes' counters alternate by launch parity), and
        // the epilogue's selection phase A goes to the token group's last slice
        if (threadIdx.x == kFinalWarp0 * 32 && (p.mode == kModeFinish || p.cs_out != nullptr)) {
          if (p.cs_out != nullptr) __threadfence();                 // the slices before their count
          const bool last = atomicAdd(fc, 1u) == 2u * p.n_ug - 1u;  // every slice of the token group written
          if (last && p.mode == kModeFinish) atomicExch(fc, 0u);
          if (p.cs_out != nullptr) *reinterpret_cast<volatile int*>(acc) = last ? 1 : 0;
        }
        if (p.cs_out != nullptr) {                                  // selection phase A (sp_score_select)
          named_bar(2, 128);
          const bool last = *reinterpret_cast<volatile int*>(acc) != 0;
          named_bar(2, 128);
          if (last) chunk_phase(p, jb, acc, tok);
          named_bar(2, 128);                                        // acc is the next job's
        }
      }
    }
  }

  // ---- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
  CHUNK_STAMP0(6);
  if (threadIdx.x == 0 && p.mode != kModeFinish) {           // finish mode never touches the partials
    // (no fence: the epoch is read by the next launch only, after this grid completes)
    if (atomicAdd(p.epoch + 1, 1u) == gridDim.x - 1) {       // last CTA: next launch uses the other buffer
      atomicExch(p.epoch + 1, 0u);
      atomicAdd(p.epoch, 1u);
    }
  }
  CHUNK_STAMP0(7);
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    cudaGetLastError();
  });
  return fn;
}

struct Plan {
  int P = 0, n_tg = 0, n_ug = 0, J = 0, T = 0, U = 0, tpc = 0, upc = 0;
  int NC = 0, NCP = 0, W = 0, nkb = 0, stages = 0, nslots = 0, swb = 0;
  long long total_jobs = 0;
  uint32_t off_k = 0, off_q = 0, off_acc = 0, off_red = 0, off_lse = 0, off_comb = 0, off_bar = 0, off_bt = 0, smem = 0;
  uint32_t k_stage_bytes = 0, q_slot_bytes = 0;
  int nq = 2;
  int hier = 0, world = 1;                            // peer exchange (world > 1); ranks
  int l2hint = 1;                                     // K tiles loaded with an L2 evict_first hint
  size_t ws_part = 0, ws_cnt = 0, ws_acc = 0, ws_fin = 0, ws_rank = 0, ws_tgr = 0;
  size_t ws_total() const { return ws_part + ws_cnt + ws_acc + ws_fin + ws_rank + ws_tgr; }
  bool ok = false;
};

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;
  }
  return n;
}

// Layout of shared memory for a given (tpc, stage count); returns total bytes.
// accpart row pitch (floats): N rounded up to 32, plus 32 -- never a power of two apart
long long acc_pitch(long long N) { return (N + 31) / 32 * 32 + 32; }

uint32_t carve(Plan& pl, int Rv, int stages) {
  uint32_t o = 0;
  pl.off_k = o;
  o += (uint32_t)stages * pl.k_stage_bytes;
  pl.off_q = o;
  o += (uint32_t)pl.nq * pl.q_slot_bytes;
  pl.off_acc = o;
  o += (uint32_t)pl.tpc * Rv * kTileM * 4;
  pl.off_red = o;
  o += 2 * 4 * pl.NCP * 8;
  pl.off_lse = o;
  o += kLseRing * pl.NCP * 4;
  o = (o + 15) & ~15u;
  pl.off_comb = o;                                   // (unused)
  pl.off_bt = o;                                     // paged K: the job's block-table slice
  o += (kMaxSlots * kTileM / 8 + 8) * 4;
  pl.off_bar = o;
  o += (2 * stages + 2 * kMaxQSlots + 2 * kMaxSlots + 4 + 2 * kLseRing) * 8 + 16;
  return o + 1024;                                   // slack for the manual 1024-byte alignment
}

// Measured plan choices (sp_score_tune / sp_score_set_plan), per geometry:
// (n_tg, n_ug, hier).
using PlanKey = std::tuple<int, int, int, int, int, int, int, long long, int, int>;
using PlanChoice = std::tuple<int, int, int, int, int>;   // (n_tg, n_ug, hier, stage cap or 0, L2 hint or -1)
std::map<PlanKey, PlanChoice>& plan_registry() {
  static std::map<PlanKey, PlanChoice> m;
  return m;
}
std::mutex& plan_registry_mu() {
  static std::mutex mu;
  return mu;
}
PlanKey plan_key(const Geom& g, int sm_budget) {
  return PlanKey(g.B, g.L, g.H, g.Hkv, g.d, g.R, g.Rv, g.N, g.esz, sm_budget);
}

// sm_budget > 0: plan for at most that many CTAs (co-scheduled peer launches on one GPU, tests).
// cands (optional): every valid (model cost, n_tg, n_ug, hier), for the tuner.
// world > 1: a peer-memory exchange over that many ranks (hier = 1).
Plan make_plan(const Geom& g, bool allow_override = true, int sm_budget = 0,
               std::vector<std::tuple<double, int, int, int>>* cands = nullptr, int world = 1) {
  Plan pl;
  pl.NC = g.G * g.Rv;
  pl.NCP = ((pl.NC + 31) / 32) * 32;                  // TMEM column groups of 32 (one tcgen05.ld.x32)
  if (pl.NCP > 16 * kMaxChunks) return pl;
  // swizzle block = the widest of 128/64/32 bytes dividing a row of d elements
  const int row_bytes = g.d * g.esz;
  if (row_bytes % 32 != 0) return pl;
  pl.swb = (row_bytes % 128 == 0) ? 128 : (row_bytes % 64 == 0 ? 64 : 32);
  pl.W = pl.swb / g.esz;
  pl.nkb = g.d / pl.W;
  pl.k_stage_bytes = (uint32_t)kTileM * row_bytes;
  pl.q_slot_bytes = (uint32_t)pl.NCP * row_bytes;
  if (pl.q_slot_bytes * 2 > 64 * 1024) return pl;
  pl.P = sm_budget > 0 ? std::min(sm_count(), sm_budget) : sm_count();
  pl.T = (int)((g.N + kTileM - 1) / kTileM);
  pl.U = g.L * g.Hkv;
  // choose (n_tg, n_ug): when a request needs more than one wave of CTAs
  // (B*J > P), J = n_tg*n_ug must divide the grid so a request never straddles
  // two waves (its CTAs exchange statistics and must be co-resident).  Time
  // model below.
  pl.nslots = std::min(kMaxSlots, kTmemCols / pl.NCP);
  double best = 1e300;
  // test/tuning override: SP_FUSED_PLAN="n_tg,n_ug[,hier]" (ignored unless valid for g)
  int force_tg = 0, force_ug = 0, force_h = -1, reg_cap = 0, reg_hint = -1;
  if (const char* env = allow_override ? std::getenv("SP_FUSED_PLAN") : nullptr) {
    const int n = std::sscanf(env, "%d,%d,%d", &force_tg, &force_ug, &force_h);
    if (n < 2) force_tg = force_ug = 0;
    if (n == 2) force_h = 0;                               // "n_tg,n_ug": the flat exchange
  }
  if (allow_override && force_tg == 0 && world == 1) {   // a measured choice for this geometry
    std::lock_guard<std::mutex> lk(plan_registry_mu());
    auto it = plan_registry().find(plan_key(g, sm_budget));
    if (it != plan_registry().end()) std::tie(force_tg, force_ug, force_h, reg_cap, reg_hint) = it->second;
  }
  pl.world = world;
  for (int J = 1; J <= pl.P; ++J) {
    if ((long long)g.B * J > pl.P && pl.P % J) continue;
    for (int n_tg = 1; n_tg <= J; ++n_tg) {
      if (J % n_tg) continue;
      const int n_ug = J / n_tg;
      if (n_tg > pl.T || n_ug > pl.U) continue;
      const int tpc = (pl.T + n_tg - 1) / n_tg, upc = (pl.U + n_ug - 1) / n_ug;
      if (tpc > pl.nslots) continue;                   // a unit's tiles must all be resident
      if (force_tg > 0 && (n_tg != force_tg || n_ug != force_ug)) continue;
      const long long jobs = (long long)g.B * J;
      const int grid = (int)std::min<long long>(pl.P, jobs);
      const long long waves = (jobs + grid - 1) / grid;
      // Time model (us, fitted to B200 measurements of C1-C4 plan sweeps): a
      // tile streams at the SM's share of HBM; a unit's lse2 is known ~L after
      // its last tile (cross-CTA skew + one L2 round trip per gather batch);
      // the TMEM ring holds W units, so L - (W-1) unit-times stay exposed; the
      // gather warp itself needs ~1.6 us per batch of kMaxLseBatch partials.
      // (per-tile costs measured for bf16 hold for e4m3 too: the statistics,
      // aggregation and exchange work per tile does not depend on the K bytes)
      const double tile_us = (double)kTileM * g.d * 2 / kSmHbmBytesPerUs;
      {
        const int hier = world > 1 ? 1 : 0;
        // single GPU: every CTA polls the unit's n_tg partials (batches of
        // kMaxLseBatch); peer: then the other ranks' words (an NVLink hop)
        const int bf = (n_tg + kMaxLseBatch - 1) / kMaxLseBatch;
        const double L_us = 5.0 + 0.8 * bf + (hier ? 2.5 : 0.0);
        const double gather_us = 1.6 * bf + (hier ? 0.2 * (world - 1) : 0.0);
        const int W = std::max(1, pl.nslots / tpc);
        const double exposed = std::max(0.0, L_us - (W - 1) * tpc * tile_us);
        // (+0.4 us fixed per unit: Q load, statistics merge and publish)
        const double per_unit = std::max(tpc * tile_us + exposed / W + 0.4, gather_us);
        double cost = upc * per_unit + L_us;                                   // + pipeline fill
        if (n_ug > 1)                                                          // cross-group max + its sync
          cost += 2.0 * g.Rv * tpc * kTileM * 4.0 / kSmHbmBytesPerUs + 5.0 + 0.25 * n_ug;
        cost *= (double)waves;
        if (cands != nullptr) cands->emplace_back(cost, n_tg, n_ug, hier);
        if (cost < best * 0.999) {
          best = cost;
          pl.J = J; pl.n_tg = n_tg; pl.n_ug = n_ug; pl.tpc = tpc; pl.upc = upc; pl.hier = hier;
        }
      }
    }
  }
  if (pl.J == 0 && force_tg > 0) return make_plan(g, false, sm_budget, nullptr, world);   // invalid override
  if (pl.J == 0) return pl;
  pl.total_jobs = (long long)g.B * pl.J;
  // 4 query slots (Q loads issued 3 units ahead) unless that costs a K stage on long units
  auto max_stages = [&](int nq) {
    pl.nq = nq;
    int s = reg_cap > 0 ? reg_cap : (world > 1 ? kStageCapPeer : kStageCap);
    while (s >= 2 && carve(pl, g.Rv, s) > (uint32_t)kSmemLimit) --s;
    return s;
  };
  const int s2 = max_stages(2), s4 = max_stages(4);
  pl.nq = (s4 >= 2 && (s4 >= s2 || pl.tpc <= 8)) ? 4 : 2;
  int stages = pl.nq == 4 ? s4 : s2;
  // development A/B knobs (timing only): SP_FUSED_NQ=2|4, SP_FUSED_MAXSTAGES=n
  if (const char* e = allow_override ? std::getenv("SP_FUSED_NQ") : nullptr) {
    const int nq = std::atoi(e);
    if ((nq == 2 && s2 >= 2) || (nq == 4 && s4 >= 2)) { pl.nq = nq; stages = nq == 4 ? s4 : s2; }
  }
  if (const char* e = allow_override ? std::getenv("SP_FUSED_MAXSTAGES") : nullptr)
    stages = std::max(2, std::min(stages, std::atoi(e)));
  if (stages < 2) return pl;
  pl.stages = stages;
  pl.smem = carve(pl, g.Rv, stages);
  pl.l2hint = reg_hint >= 0 ? reg_hint : 1;
  if (const char* e = allow_override ? std::getenv("SP_FUSED_L2HINT") : nullptr) pl.l2hint = std::atoi(e) != 0;
  pl.ws_part = align256(2 * (size_t)g.B * pl.U * pl.NCP * pl.n_tg * sizeof(unsigned long long));
  pl.ws_cnt = 256;                                   // launch epoch + CTAs-done counter
  pl.ws_acc = pl.n_ug > 1 ? align256((size_t)g.B * pl.n_ug * g.Rv * acc_pitch(g.N) * sizeof(float)) : 0;
  pl.ws_fin = align256((size_t)3 * g.B * pl.n_tg * sizeof(unsigned));
  pl.ws_rank = 0;
  pl.ws_tgr = align256((size_t)g.B * pl.n_tg * sizeof(unsigned));   // token-group boundary counters (sp_score_select)
  pl.ok = true;
  return pl;
}

bool encode_maps(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay, const Plan& pl,
                 CUtensorMap* tmK, CUtensorMap* tmQ) {
  PFN_encodeTiled_t enc = encode_fn();
  if (enc == nullptr) return false;
  const CUtensorMapSwizzle sw = pl.swb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                               : (pl.swb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  const CUtensorMapDataType dt = g.esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const long long esz = g.esz;
  // strides of size-1 dims are irrelevant; give them a harmless contiguous value
  auto fix = [esz](long long stride, long long prev_extent_bytes, long long size) -> cuuint64_t {
    return (size == 1 || stride == 0) ? (cuuint64_t)prev_extent_bytes : (cuuint64_t)(stride * esz);
  };
  {
    cuuint64_t dims[5] = {(cuuint64_t)g.d, (cuuint64_t)g.N, (cuuint64_t)g.Hkv, (cuuint64_t)g.L, (cuuint64_t)g.B};
    cuuint64_t s1 = fix(lay.k_i, (long long)g.d * esz, g.N);
    cuuint64_t s2 = fix(lay.k_g, (long long)s1 * g.N, g.Hkv);
    cuuint64_t s3 = fix(lay.k_l, (long long)s2 * g.Hkv, g.L);
    cuuint64_t s4 = fix(lay.k_b, (long long)s3 * g.L, g.B);
    cuuint64_t strides[4] = {s1, s2, s3, s4};
    cuuint32_t box[5] = {(cuuint32_t)pl.W, (cuuint32_t)kTileM, 1, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (enc(tmK, dt, 5, const_cast<__nv_bfloat16*>(K), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  {
    cuuint64_t dims[5] = {(cuuint64_t)g.d, (cuuint64_t)g.H, (cuuint64_t)g.R, (cuuint64_t)g.L, (cuuint64_t)g.B};
    cuuint64_t s1 = fix(lay.q_h, (long long)g.d * esz, g.H);
    cuuint64_t s2 = fix(lay.q_r, (long long)s1 * g.H, g.R);
    cuuint64_t s3 = fix(lay.q_l, (long long)s2 * g.R, g.L);
    cuuint64_t s4 = fix(lay.q_b, (long long)s3 * g.L, g.B);
    cuuint64_t strides[4] = {s1, s2, s3, s4};
    cuuint32_t box[5] = {(cuuint32_t)pl.W, (cuuint32_t)g.G, (cuuint32_t)g.Rv, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (enc(tmQ, dt, 5, const_cast<__nv_bfloat16*>(Q), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

}  // namespace

#ifdef SP_CHUNK_TRACE
extern "C" int sp_chunk_trace_read(unsigned long long* host, int reset) {   // [160][8]
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(host, g_chunk_trace, sizeof(g_chunk_trace)) != cudaSuccess) return 1;
  if (reset) {
    static unsigned long long z[160][8] = {};
    if (cudaMemcpyToSymbol(g_chunk_trace, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}
#endif

static unsigned long long* g_trace = nullptr;
static long long g_trace_records = 0;

void fused_set_trace(unsigned long long* buf, long long records) {
  g_trace = buf;
  g_trace_records = records;
}

bool fused_supported(const Geom& g, const Layout&, const void*, const void*) {
  if (g.G > 256 || g.Rv > 256) return false;         // TMA box dims
  return make_plan(g).ok;
}

bool fused_plan_info(const Geom& g, long long out[kPlanInfo]) {
  Plan pl = make_plan(g);
  if (!pl.ok) return false;
  out[0] = std::min<long long>(pl.P, pl.total_jobs); out[1] = pl.J; out[2] = pl.n_tg; out[3] = pl.n_ug;
  out[4] = pl.tpc; out[5] = pl.upc; out[6] = pl.nslots; out[7] = pl.stages; out[8] = pl.smem; out[9] = pl.hier;
  return true;
}

size_t fused_score_ws_bytes(const Geom& g) {
  Plan pl = make_plan(g);
  if (!pl.ok) return 0;
  return pl.ws_total();
}

namespace {

// Stats-only mode epilogue: merge each unit's n_tg CTA partials (buffer of the
// launch that just ran: its parity is epoch - 1) into per-row (m2, l) in the
// sp_score_stats layout, row = ((b*L + l)*H + h)*Rv + r.
__global__ void k_partials_to_stats(const unsigned long long* __restrict__ part, const unsigned* __restrict__ epoch,
                                    int B, int L, int Hkv, int G, int Rv, int n_tg, int NC, int NCP,
                                    float* __restrict__ stats) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long U = (long long)L * Hkv;
  if (idx >= (long long)B * U * NC) return;
  const int c = (int)(idx % NC);
  const long long ubase = idx / NC;                  // b*U + u
  const int u = (int)(ubase % U), b = (int)(ubase / U);
  const int l = u / Hkv, g = u % Hkv;
  const unsigned parity = (epoch[0] - 1u) & 1u;
  const long long half = (long long)B * U * n_tg * NCP;
  const unsigned long long* src = part + parity * half + ubase * n_tg * NCP + c;
  float M = -CUDART_INF_F, S = 0.f;
  for (int s2 = 0; s2 < n_tg; ++s2) {
    const float2 w = unpack_ms(src[(long long)s2 * NCP]);
    if (w.y > 0.f) merge2(M, S, w.x, w.y);
  }
  const long long row = (((long long)b * L + l) * Hkv * G + g * G + c % G) * Rv + c / G;
  stats[row * 2] = M;
  stats[row * 2 + 1] = S;
}

}  // namespace

struct DeferOut {
  const float* accp = nullptr;                        // [B][n_ug][Rv][pitch] partial maps (in the workspace)
  long long pitch = 0;
  int n_ug = 0;
};

struct PeerArgs {
  int rank = 0, world = 1, sm_budget = 0;
  void* const* bufs = nullptr;                        // world partial buffers (fused_peer_buffer_bytes each)
};

// The epilogue's selection phase A needs the token group's importance plus the
// pooling halo and its pooled values staged in the acc region (tpc * Rv * 128
// floats), whole chunks in the selection kernel's segments (chunk <= 16384), and
// a plain single-GPU importance launch.
bool chunk_phase_fits(const Geom& g, const Plan& pl, int mode, const float* acc_out, int world, const PagedK* pk,
                      int pool_k, int chunk) {
  if (mode != kModeFull || acc_out != nullptr || world != 1 || chunk < 1 || chunk > 16384 || pool_k < 1) return false;
  if (pk != nullptr && pk->seq_lens != nullptr) return false;
  const long long w = (pool_k - 1) / 2;
  // no chunk's windows may cross both boundaries of a token group
  if (pl.n_tg >= 3 && (long long)(pl.T / pl.n_tg) * kTileM < 2 * (w + chunk)) return false;
  const long long span = (long long)pl.tpc * kTileM + 2 * (chunk + w);   // pooled tokens, at most
  const long long need = ((span + 2 * w + 3) & ~3LL) + span;
  return need <= (long long)pl.tpc * g.Rv * kTileM;
}

// Row f3: the paged-cache tensor map {d, Hkv, block_size, blocks, L}, box {W, 1, min(bs, 128), 1, 1}.
bool encode_paged_map(const PagedK& pk, const Geom& g, const Plan& pl, CUtensorMap* tmK) {
  PFN_encodeTiled_t enc = encode_fn();
  if (enc == nullptr) return false;
  const CUtensorMapSwizzle sw = pl.swb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                               : (pl.swb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  const CUtensorMapDataType dt = g.esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const long long esz = g.esz;
  auto fix = [esz](long long stride, long long prev_extent_bytes, long long size) -> cuuint64_t {
    return (size == 1 || stride == 0) ? (cuuint64_t)prev_extent_bytes : (cuuint64_t)(stride * esz);
  };
  cuuint64_t dims[5] = {(cuuint64_t)g.d, (cuuint64_t)g.Hkv, (cuuint64_t)pk.bs, (cuuint64_t)pk.num_blocks,
                        (cuuint64_t)g.L};
  cuuint64_t s1 = fix(pk.s_g, (long long)g.d * esz, g.Hkv);
  cuuint64_t s2 = fix(pk.s_tok, (long long)s1 * g.Hkv, pk.bs);
  cuuint64_t s3 = fix(pk.s_blk, (long long)s2 * pk.bs, pk.num_blocks);
  cuuint64_t s4 = fix(pk.s_l, (long long)s3 * pk.num_blocks, g.L);
  cuuint64_t strides[4] = {s1, s2, s3, s4};
  cuuint32_t box[5] = {(cuuint32_t)pl.W, 1, (cuuint32_t)std::min(pk.bs, kTileM), 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return enc(tmK, dt, 5, const_cast<void*>(pk.cache), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row f3, block_size < 128: one box per block covering all of d.  The tensor map
// splits a block's rows into (row_lo = 8, row_hi = bs/8) and d into (W, nkb) with
// dims {W, row_lo, nkb, row_hi, idx}, so the box lands as [row_hi][kb][8 rows][W]:
// 8-row groups with their kb halves adjacent (the A operand's group stride is
// nkb * 1024 B).  idx = (l*s_l + blk*s_blk + g*s_g) / s_g addresses a block row
// span of one kv head, so the layer and block strides must be multiples of s_g.
// Returns false (caller uses the two-box-per-block map) when the strides do not
// fold, nkb < 2, the swizzle is not 128 B or the driver rejects the map.
bool encode_paged_interleaved(const PagedK& pk, const Geom& g, const Plan& pl, CUtensorMap* tmK, int* fl, int* fb) {
  if (pl.nkb < 2 || pl.swb != 128 || pk.s_g <= 0 || pk.bs < 8) return false;
  if (pk.s_l % pk.s_g != 0 || pk.s_blk % pk.s_g != 0) return false;
  const long long FL = pk.s_l / pk.s_g, FB = pk.s_blk / pk.s_g;
  const long long extent = (long long)(g.L - 1) * FL + (long long)(pk.num_blocks - 1) * FB + g.Hkv;
  if (extent >= (1LL << 31) || FL >= (1LL << 31) || FB >= (1LL << 31)) return false;
  PFN_encodeTiled_t enc = encode_fn();
  if (enc == nullptr) return false;
  const long long esz = g.esz;
  cuuint64_t dims[5] = {(cuuint64_t)pl.W, 8, (cuuint64_t)pl.nkb, (cuuint64_t)(pk.bs / 8), (cuuint64_t)extent};
  cuuint64_t strides[4] = {(cuuint64_t)(pk.s_tok * esz), (cuuint64_t)pl.swb, (cuuint64_t)(8 * pk.s_tok * esz),
                           (cuuint64_t)(pk.s_g * esz)};
  cuuint32_t box[5] = {(cuuint32_t)pl.W, 8, (cuuint32_t)pl.nkb, (cuuint32_t)(pk.bs / 8), 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUtensorMapDataType dt = g.esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (enc(tmK, dt, 5, const_cast<void*>(pk.cache), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return false;
  *fl = (int)FL;
  *fb = (int)FB;
  return true;
}

cudaError_t fused_launch(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay, int mode,
                         const float* lse_in, float* importance, void* ws, size_t ws_bytes, cudaStream_t st,
                         float* acc_out = nullptr, const PeerArgs& peer = PeerArgs(), const PagedK* pk = nullptr,
                         const float2* la = nullptr, const ChunkOut* co = nullptr, DeferOut* dfr = nullptr) {
  if (peer.world < 1 || peer.world > kMaxPeers || peer.rank < 0 || peer.rank >= peer.world) return cudaErrorInvalidValue;
  Plan pl = make_plan(g, true, peer.sm_budget, nullptr, peer.world);
  if (!pl.ok || ws_bytes < pl.ws_total()) return cudaErrorInvalidValue;
  if (peer.world > 1 && (peer.bufs == nullptr || !pl.hier)) return cudaErrorInvalidValue;
  static FusedParams p;                               // large (two tensor maps); host-side scratch
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  std::memset(&p, 0, sizeof(p));
  if (!encode_maps(Q, K, g, lay, pl, &p.tmK, &p.tmQ)) return cudaErrorInvalidValue;
  if (pk != nullptr) {
    int fl = 0, fb = 0;
    if (pk->bs < kTileM && encode_paged_interleaved(*pk, g, pl, &p.tmK, &fl, &fb)) {
      p.kinter = 1;
      p.fl = fl;
      p.fb = fb;
    } else if (!encode_paged_map(*pk, g, pl, &p.tmK)) {
      return cudaErrorInvalidValue;
    }
    p.paged = 1;
    p.bs = pk->bs;
    p.bs_log2 = __builtin_ctz((unsigned)pk->bs);
    p.btab = pk->btab;
    p.max_blocks = pk->max_blocks;
    p.seq_lens = pk->seq_lens;
  }
  p.B = g.B; p.L = g.L; p.Hkv = g.Hkv; p.G = g.G; p.Rv = g.Rv; p.d = g.d; p.N = (int)g.N;
  p.T = pl.T; p.U = pl.U; p.n_tg = pl.n_tg; p.n_ug = pl.n_ug; p.J = pl.J; p.total_jobs = pl.total_jobs;
  p.NC = pl.NC; p.NCP = pl.NCP; p.W = pl.W; p.nkb = pl.nkb; p.stages = pl.stages; p.nslots = pl.nslots;
  p.tpc = pl.tpc;
  p.esz = g.esz; p.swb = pl.swb; p.ksteps = pl.swb / 32;
  p.xs = g.scale * kLog2e;
  // instruction descriptor: D fp32 (bit 4); A/B format bf16 (1) for kind::f16,
  // e4m3 (0) for kind::f8f6f4; K-major A and B; N >> 3 at bit 17, M >> 4 at bit 24
  const uint32_t ab_fmt = g.esz == 2 ? ((1u << 7) | (1u << 10)) : 0u;
  p.idesc = (1u << 4) | ab_fmt | ((uint32_t)(pl.NCP >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);
  p.layout_type = pl.swb == 128 ? 2u : (pl.swb == 64 ? 4u : 6u);
  p.off_k = pl.off_k; p.off_q = pl.off_q; p.off_acc = pl.off_acc; p.off_red = pl.off_red; p.off_lse = pl.off_lse; p.off_comb = pl.off_comb;
  p.off_bar = pl.off_bar; p.off_bt = pl.off_bt; p.k_stage_bytes = pl.k_stage_bytes; p.q_slot_bytes = pl.q_slot_bytes;
  p.nq = pl.nq;
  char* w = reinterpret_cast<char*>(ws);
  // counters first: their offsets depend only on (B, U), not on the plan
  p.epoch = reinterpret_cast<unsigned*>(w);
  w += pl.ws_cnt;
  p.fin_cnt = reinterpret_cast<unsigned*>(w);
  w += pl.ws_fin;
  p.part = reinterpret_cast<unsigned long long*>(w);
  w += pl.ws_part;
  p.accpart = pl.ws_acc ? reinterpret_cast<float*>(w) : nullptr;
  p.acc_pitch = acc_pitch(g.N);
  w += pl.ws_acc;
  p.bnd_cnt = reinterpret_cast<unsigned*>(w);
  w += pl.ws_tgr;
  if (co != nullptr) {
    if (!chunk_phase_fits(g, pl, mode, acc_out, peer.world, pk, co->pool_k, co->chunk)) return cudaErrorNotSupported;
    p.cs_out = co->cs;
    p.pool_k = co->pool_k;
    p.chunk = co->chunk;
    p.n_c_row = (g.N + co->chunk - 1) / co->chunk;
  }
  if (dfr != nullptr) {
    if (pl.n_ug < 2 || p.accpart == nullptr || co != nullptr) return cudaErrorNotSupported;
    p.defer = 1;
    dfr->accp = p.accpart;
    dfr->pitch = p.acc_pitch;
    dfr->n_ug = pl.n_ug;
  }
  p.hier = pl.hier;
  p.rank = peer.rank;
  p.world = peer.world;
  if (peer.world > 1) {
    for (int r = 0; r < peer.world; ++r) p.peer[r] = reinterpret_cast<unsigned long long*>(peer.bufs[r]);
  }
  p.imp = importance;
  p.acc_out = acc_out;
  p.l2hint = pl.l2hint;
  p.err = device_error_flag();
  p.trace = nullptr;
  p.mode = mode;
  p.lse_in = lse_in;
  p.la = la;

  p.trace_units = 0;
  if (g_trace != nullptr) {
    const long long grid = std::min<long long>(pl.P, pl.total_jobs);
    const long long tail = g_trace_records > 16000 ? 8000 : 0;   // (trace builds only)   // per-tile stamps of CTA 0 at the end
    const long long units = ((g_trace_records - tail) / 8) / grid;
    if (units > 0) {
      p.trace = g_trace;
      p.tile_trace = tail ? g_trace + g_trace_records - tail : nullptr;
      p.trace_units = (int)std::min<long long>(units, 1 << 30);
    }
  }

  // one instantiation per (GQA group, one-column-group, input type)
  using KernFn = void (*)(FusedParams);
  static const KernFn table[2][5][2] = {
      {{k_fused<1, 0, false>, k_fused<1, 32, false>}, {k_fused<2, 0, false>, k_fused<2, 32, false>},
       {k_fused<4, 0, false>, k_fused<4, 32, false>}, {k_fused<8, 0, false>, k_fused<8, 32, false>},
       {k_fused<0, 0, false>, k_fused<0, 32, false>}},
      {{k_fused<1, 0, true>, k_fused<1, 32, true>}, {k_fused<2, 0, true>, k_fused<2, 32, true>},
       {k_fused<4, 0, true>, k_fused<4, 32, true>}, {k_fused<8, 0, true>, k_fused<8, 32, true>},
       {k_fused<0, 0, true>, k_fused<0, 32, true>}}};
  // the >48 KiB dynamic-SMEM opt-in is per device: set once per (device, instantiation)
  static bool configured[64][2][5][2] = {};
  const int kt = g.esz == 1 ? 1 : 0;
  const int ki = g.G == 1 ? 0 : g.G == 2 ? 1 : g.G == 4 ? 2 : g.G == 8 ? 3 : 4;
  const int kj = pl.NCP == 32 ? 1 : 0;
  KernFn kern = table[kt][ki][kj];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!configured[dev][kt][ki][kj]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e != cudaSuccess) return e;
    configured[dev][kt][ki][kj] = true;
  }
  const int grid = (int)std::min<long long>(pl.P, pl.total_jobs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;       // all CTAs co-resident (in-kernel exchange)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t fused_score(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                        float* importance, void* ws, size_t ws_bytes, cudaStream_t st) {
  return fused_launch(Q, K, g, lay, kModeFull, nullptr, importance, ws, ws_bytes, st);
}

cudaError_t fused_score_deferred(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                                 void* ws, size_t ws_bytes, cudaStream_t st, const float** accp, int* n_ug,
                                 long long* pitch) {
  Plan pl = make_plan(g);
  if (!pl.ok || pl.n_ug < 2) return cudaErrorNotSupported;          // nothing to defer: one unit group
  DeferOut d;
  const cudaError_t e = fused_launch(Q, K, g, lay, kModeFull, nullptr, nullptr, ws, ws_bytes, st, nullptr, PeerArgs(),
                                     nullptr, nullptr, nullptr, &d);
  if (e == cudaSuccess) {
    *accp = d.accp;
    *n_ug = d.n_ug;
    *pitch = d.pitch;
  }
  return e;
}

cudaError_t fused_score_chunks(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                               float* importance, const ChunkOut& co, void* ws, size_t ws_bytes, cudaStream_t st) {
  return fused_launch(Q, K, g, lay, kModeFull, nullptr, importance, ws, ws_bytes, st, nullptr, PeerArgs(), nullptr,
                      nullptr, &co);
}

// Z2' (row f4): the look-ahead keys' (max2, sum) per (request, unit, column), one
// warp per (b, l, h, r): x_j = xs * <Q[b][l][r][h], K_la[b][l][h/G][j]> for
// j <= r - shift (fp32 FMA of exact bf16 products), log2 domain.
__global__ void k_la_stats(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Kla, Layout lay,
                           LookaheadK la, int B, int L, int H, int Hkv, int Rv, int d, int NCP, float xs,
                           float2* __restrict__ out) {
  const long long row = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= (long long)B * L * H * Rv) return;
  const int r = (int)(row % Rv), h = (int)((row / Rv) % H), l = (int)((row / ((long long)Rv * H)) % L);
  const int b = (int)(row / ((long long)Rv * H * L));
  const int G = H / Hkv, g = h / G;
  const __nv_bfloat16* q = Q + b * lay.q_b + l * lay.q_l + r * lay.q_r + h * lay.q_h;
  float qv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) qv[k] = lane + 32 * k < d ? __bfloat162float(q[lane + 32 * k]) : 0.f;
  float m = -CUDART_INF_F, s = 0.f;
  const int n_la = r + 1 - la.shift;
  for (int j = 0; j < n_la; ++j) {
    const __nv_bfloat16* kr = Kla + b * la.s_b + l * la.s_l + g * la.s_g + j * la.s_j;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (lane + 32 * k < d) acc = fmaf(qv[k], __bfloat162float(kr[lane + 32 * k]), acc);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    merge2(m, s, acc * xs, 1.f);
  }
  if (lane == 0) out[((long long)b * L * Hkv + (long long)l * Hkv + g) * NCP + r * G + (h % G)] = make_float2(m, s);
}

size_t fused_la_ws_bytes(const Geom& g) {
  const size_t base = fused_score_ws_bytes(g);
  if (base == 0) return 0;
  const int NCP = ((g.G * g.Rv + 31) / 32) * 32;
  return align256(base) + align256((size_t)g.B * g.L * g.Hkv * NCP * sizeof(float2));
}

cudaError_t fused_score_la(const __nv_bfloat16* Q, const __nv_bfloat16* K, const LookaheadK& la, const Geom& g,
                           const Layout& lay, float* importance, void* ws, size_t ws_bytes, cudaStream_t st) {
  const size_t base = align256(fused_score_ws_bytes(g));
  if (base == 0 || ws_bytes < fused_la_ws_bytes(g)) return cudaErrorInvalidValue;
  const int NCP = ((g.G * g.Rv + 31) / 32) * 32;
  float2* lab = reinterpret_cast<float2*>(reinterpret_cast<char*>(ws) + base);
  const long long rows = (long long)g.B * g.L * g.H * g.Rv;
  k_la_stats<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(Q, reinterpret_cast<const __nv_bfloat16*>(la.K), lay, la,
                                                         g.B, g.L, g.H, g.Hkv, g.Rv, g.d, NCP, g.scale * kLog2e, lab);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return fused_launch(Q, K, g, lay, kModeFull, nullptr, importance, ws, base, st, nullptr, PeerArgs(), nullptr, lab);
}

cudaError_t fused_score_paged(const __nv_bfloat16* Q, const PagedK& K, const Geom& g, const Layout& lay,
                              float* importance, void* ws, size_t ws_bytes, cudaStream_t st) {
  Layout l2 = lay;
  l2.k_b = l2.k_l = l2.k_g = l2.k_i = 0;                    // (the contiguous map is replaced by the paged one)
  return fused_launch(Q, reinterpret_cast<const __nv_bfloat16*>(K.cache), g, l2, kModeFull, nullptr, importance, ws,
                      ws_bytes, st, nullptr, PeerArgs(), &K);
}

// Measured plan choice (sp_score_tune): the model's best candidates (cost within
// 1.3x, at most 6) each timed over 5 launches on private zeroed workspaces; the
// fastest is registered for g and used by every later plan query of g.
#ifndef SP_TUNE_MAX
#define SP_TUNE_MAX 6
#endif
#ifndef SP_TUNE_SPAN
#define SP_TUNE_SPAN 1.3
#endif
constexpr int kTuneMax = SP_TUNE_MAX;        // candidates timed
constexpr double kTuneSpan = SP_TUNE_SPAN;   // ... within this factor of the model's best cost
cudaError_t fused_tune(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                       cudaStream_t user_st, int* tg_out, int* ug_out, int* hier_out, float* ms_out) {
  constexpr int kReps = 10;
  std::vector<std::tuple<double, int, int, int>> cands;
  {
    std::lock_guard<std::mutex> lk(plan_registry_mu());
    plan_registry().erase(plan_key(g, 0));
  }
  Plan base = make_plan(g, false, 0, &cands);
  if (!base.ok) return cudaErrorInvalidValue;
  // a private stream (capturable, unlike the legacy default stream), ordered after the caller's
  cudaStream_t st = nullptr;
  cudaEvent_t ready = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return cudaGetLastError();
  if (cudaEventCreate(&ready) != cudaSuccess) {
    cudaStreamDestroy(st);
    return cudaGetLastError();
  }
  cudaEventRecord(ready, user_st);
  cudaStreamWaitEvent(st, ready, 0);
  std::sort(cands.begin(), cands.end());
  const double best_cost = std::get<0>(cands.front());
  float best_ms = 1e30f;
  int best_tg = base.n_tg, best_ug = base.n_ug, best_h = base.hier, best_cap = 0, best_hint = -1;
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return cudaGetLastError();
  float* imp = nullptr;
  cudaError_t err = cudaMalloc(&imp, (size_t)g.B * g.N * sizeof(float));
  for (size_t i = 0; err == cudaSuccess && i < cands.size() && i < (size_t)kTuneMax; ++i) {
    if (std::get<0>(cands[i]) > kTuneSpan * best_cost) break;
    const int tg = std::get<1>(cands[i]), ug = std::get<2>(cands[i]), h = std::get<3>(cands[i]);
    int last_stages = -1;
    for (int hint : {1, 0})                                        // L2 evict_first on the K stream, or not
    for (int cap : {kStageCap, kStageCap - 1}) {                 // (measured: 3 or 4 TMA stages win)
      if (cap == kStageCap) last_stages = -1;
      {
        std::lock_guard<std::mutex> lk(plan_registry_mu());
        plan_registry()[plan_key(g, 0)] = PlanChoice(tg, ug, h, cap, hint);
      }
      Plan pl = make_plan(g);
      if (!pl.ok || pl.n_tg != tg || pl.n_ug != ug || pl.hier != h || pl.stages == last_stages) continue;
      last_stages = pl.stages;
      void* ws = nullptr;
      if ((err = cudaMalloc(&ws, pl.ws_total())) != cudaSuccess) break;
      cudaMemsetAsync(ws, 0, pl.ws_total(), st);
      for (int w = 0; w < 2 && err == cudaSuccess; ++w) err = fused_score(Q, K, g, lay, imp, ws, pl.ws_total(), st);
      // kReps launches replayed as a CUDA graph: the host's per-launch preparation
      // (plan, tensor maps) must not pace short kernels (a 4K prompt runs ~60 us)
      float ms = 1e30f;
      cudaGraph_t graph = nullptr;
      cudaGraphExec_t exec = nullptr;
      if (err == cudaSuccess) err = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      if (err == cudaSuccess) {
        cudaError_t e2 = cudaSuccess;
        for (int r = 0; r < kReps && e2 == cudaSuccess; ++r) e2 = fused_score(Q, K, g, lay, imp, ws, pl.ws_total(), st);
        err = cudaStreamEndCapture(st, &graph);
        if (err == cudaSuccess) err = e2;
      }
      if (err == cudaSuccess) err = cudaGraphInstantiate(&exec, graph, 0);
      for (int it = 0; it < 4 && err == cudaSuccess; ++it) {       // first replay warms up
        cudaEventRecord(e0, st);
        err = cudaGraphLaunch(exec, st);
        cudaEventRecord(e1, st);
        if (err == cudaSuccess) err = cudaEventSynchronize(e1);
        float t = 0.f;
        if (err == cudaSuccess && it > 0 && cudaEventElapsedTime(&t, e0, e1) == cudaSuccess) ms = std::min(ms, t);
      }
      if (exec != nullptr) cudaGraphExecDestroy(exec);
      if (graph != nullptr) cudaGraphDestroy(graph);
      cudaStreamSynchronize(st);
      cudaFree(ws);
      // the model's plan (timed first) is kept unless a candidate beats it by
      // more than the timing noise (about 1 %: a graph of 10 launches)
      if (err == cudaSuccess && ms < best_ms * (best_ms < 1e29f ? 0.99f : 1.f)) {
        best_ms = ms; best_tg = tg; best_ug = ug; best_h = h; best_cap = cap; best_hint = hint;
      }
    }
  }
  cudaStreamSynchronize(st);
  cudaFree(imp);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(ready);
  cudaStreamDestroy(st);
  {
    std::lock_guard<std::mutex> lk(plan_registry_mu());
    plan_registry()[plan_key(g, 0)] = PlanChoice(best_tg, best_ug, best_h, best_cap, best_hint);
  }
  *tg_out = best_tg;
  *ug_out = best_ug;
  *hier_out = best_h;
  *ms_out = best_ms / kReps;
  return err;
}

bool fused_set_plan(const Geom& g, int n_tg, int n_ug, int hier) {
  std::lock_guard<std::mutex> lk(plan_registry_mu());
  if (n_tg <= 0) { plan_registry().erase(plan_key(g, 0)); return true; }
  plan_registry()[plan_key(g, 0)] = PlanChoice(n_tg, n_ug, hier, 0, -1);
  return true;
}

cudaError_t fused_score_stats(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                              float* stats, void* ws, size_t ws_bytes, cudaStream_t st) {
  cudaError_t e = fused_launch(Q, K, g, lay, kModeStats, nullptr, nullptr, ws, ws_bytes, st);
  if (e != cudaSuccess) return e;
  Plan pl = make_plan(g);
  const char* w = reinterpret_cast<const char*>(ws);
  const unsigned* epoch = reinterpret_cast<const unsigned*>(w);
  const unsigned long long* part = reinterpret_cast<const unsigned long long*>(w + pl.ws_cnt + pl.ws_fin);
  const long long n = (long long)g.B * pl.U * pl.NC;
  k_partials_to_stats<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, epoch, g.B, g.L, g.Hkv, g.G, g.Rv, pl.n_tg,
                                                                   pl.NC, pl.NCP, stats);
  return cudaGetLastError();
}

cudaError_t fused_score_finish(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                               const float* lse2, float* importance, void* ws, size_t ws_bytes, cudaStream_t st) {
  return fused_launch(Q, K, g, lay, kModeFinish, lse2, importance, ws, ws_bytes, st);
}

cudaError_t fused_score_acc(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                            float* acc2, void* ws, size_t ws_bytes, cudaStream_t st) {
  return fused_launch(Q, K, g, lay, kModeFull, nullptr, nullptr, ws, ws_bytes, st, acc2);
}

size_t fused_peer_buffer_bytes(const Geom& g, int world, int sm_budget) {
  Plan pl = make_plan(g, true, sm_budget, nullptr, world);
  if (!pl.ok) return 0;
  return align256(2 * (size_t)g.B * pl.U * pl.NCP * world * sizeof(unsigned long long));   // rank words
}

size_t fused_peer_ws_bytes(const Geom& g, int world, int sm_budget) {
  Plan pl = make_plan(g, true, sm_budget, nullptr, world);
  return pl.ok ? pl.ws_total() : 0;
}

bool fused_peer_plan_info(const Geom& g, int world, int sm_budget, long long out[kPlanInfo]) {
  Plan pl = make_plan(g, true, sm_budget, nullptr, world);
  if (!pl.ok) return false;
  out[0] = std::min<long long>(pl.P, pl.total_jobs); out[1] = pl.J; out[2] = pl.n_tg; out[3] = pl.n_ug;
  out[4] = pl.tpc; out[5] = pl.upc; out[6] = pl.nslots; out[7] = pl.stages; out[8] = pl.smem; out[9] = pl.hier;
  return true;
}

cudaError_t fused_score_peer(const __nv_bfloat16* Q, const __nv_bfloat16* K, const Geom& g, const Layout& lay,
                             int rank, int world, void* const* bufs, int sm_budget, float* importance, void* ws,
                             size_t ws_bytes, cudaStream_t st) {
  PeerArgs pa;
  pa.rank = rank;
  pa.world = world;
  pa.bufs = bufs;
  pa.sm_budget = sm_budget;
  return fused_launch(Q, K, g, lay, kModeFull, nullptr, importance, ws, ws_bytes, st, nullptr, pa);
}

namespace {
// imp[b][i] = (1/Rv) sum_{r<Rv} 2^acc2[b][r][i] -- the fused epilogue's arithmetic,
// applied after the head-sharded max-reduce.
__global__ void k_acc_importance(const float* __restrict__ acc2, int B, int Rv, long long N, float* __restrict__ imp) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * N) return;
  const long long b = idx / N, i = idx % N;
  float s = 0.f;
  for (int r = 0; r < Rv; ++r) s += ex2(acc2[(b * Rv + r) * N + i]);
  imp[idx] = s * (1.f / (float)Rv);
}
}  // namespace

cudaError_t acc_importance(const float* acc2, int B, int Rv, long long N, float* importance, cudaStream_t st) {
  const long long n = (long long)B * N;
  k_acc_importance<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(acc2, B, Rv, N, importance);
  return cudaGetLastError();
}

}  // namespace sp
