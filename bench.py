#!/usr/bin/env python
"""Bench of the SpecPrefill hot path on B200: prompt tokens scored+selected/s.

One step = sp_score -> sp_select -> sp_gather over one batch of synthetic
input already resident in HBM (the whole hot path, SURVEY.md §8(a) rows
a1-a11).  Default workload: BASELINE.json configs[3] (8B-shaped speculator,
32K prompt, keep 10%) -- the configuration the north_star's >=70%-of-HBM
target is quoted on.  K (2 GiB) is far larger than L2 (126 MB), so no L2
flush is needed between steps.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--algo fused|simt]
  python bench.py --impl reference ...     # the float64 oracle on host cores (the reference arm)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prompt tokens scored+selected/sec"
UNIT = "tokens/s"
HBM_FALLBACK_GBS = 6650.0           # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)
SPEC_HBM_GBS = 8000.0               # BASELINE.json "~8 TB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=["C0", "C1", "C2", "C3", "C4"])
    ap.add_argument("--R", type=int, default=None, help="secondary point: look-ahead rows (SURVEY 8(d): R=1 'Full', R=9)")
    ap.add_argument("--chunk", type=int, default=None, help="secondary point: chunk size (chunk=1: raw SpecPrefill)")
    ap.add_argument("--pool", type=int, default=None, help="secondary point: pooling window (odd)")
    ap.add_argument("--keep", type=float, default=None, help="secondary point: keep rate")
    ap.add_argument("--algo", default="fused", choices=["fused", "simt", "auto"])
    ap.add_argument("--plan", default=None, help="fused-kernel decomposition override 'n_tg,n_ug'")
    ap.add_argument("--shard", default="auto", choices=["auto", "batch", "replica", "seq", "seq-split", "head"],
                    help="N>1: batch = the batch's requests split over ranks (dist.batch_range), no collective "
                         "(strong scaling); replica = every rank runs its own copy of the workload (weak); "
                         "seq = the prompt split over ranks, statistics exchanged inside the fused kernel over "
                         "NVLink peer memory (one K read) + the sharded selection (candidate all-gather/merge; "
                         "strong); seq-split = the same split with stats/finish launches and an NCCL statistics "
                         "all-gather (two K reads); head = the heads split over ranks, NCCL MAX all-reduce of the "
                         "log-domain maxima (strong).  auto: C2 -> batch, C3/C4 -> seq (BASELINE.json configs), "
                         "C0/C1 -> replica")
    ap.add_argument("--kv", default="bf16", choices=["bf16", "e4m3"],
                    help="input element type: bf16 (the north_star's), or e4m3 codes with per-tensor scales "
                         "(SURVEY 8(f) row f4, sp_score_e4m3; single GPU / batch sharding)")
    ap.add_argument("--paged", type=int, default=0, metavar="BS",
                    help="K in a paged cache of block size BS with a shuffled block table (row f3, sp_score_paged)")
    ap.add_argument("--paged-layout", default="hnd", choices=["hnd", "nhd"],
                    help="block storage: hnd = [Hkv][BS][d] per block (a head's rows contiguous), "
                         "nhd = [BS][Hkv][d] (heads interleaved per token)")
    ap.add_argument("--ragged", action="store_true",
                    help="with --paged: per-request prompt lengths uniform in [N/4, N] (seeded); tokens/s counts "
                         "the real tokens")
    ap.add_argument("--no-tune", action="store_true",
                    help="skip sp_score_tune (the fused plan measured among the model's best candidates during "
                         "warm-up, untimed); single-GPU / batch-sharded contiguous inputs only")
    ap.add_argument("--two-launch", action="store_true",
                    help="A/B: sp_score (with its cross-unit-group epilogue) then sp_select_gather, instead of "
                         "sp_score_select (the selection finalizes the importance)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly instead of replaying a CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-read-peak", action="store_true", help="skip measuring the read-only stream peak")
    ap.add_argument("--cpu-sample-layers", type=int, default=32)
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        busy = [s for s in sm if s > 0.5 * max(sm)]
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


_SECONDARY = {}


def workload(name):
    """BASELINE.json config `name`, with the secondary-point overrides of SURVEY
    8(d) (--R, --chunk, --pool, --keep) if given."""
    from spgen import gen
    w = gen.CONFIGS[name]
    kw = {k: v for k, v in _SECONDARY.items() if v is not None}
    return w.with_(**kw) if kw else w


def secondary_label() -> str:
    kw = {k: v for k, v in _SECONDARY.items() if v is not None}
    return (" (" + ", ".join(f"{k}={v}" for k, v in kw.items()) + ")") if kw else ""


def kept_chunks_tokens(w) -> int:
    """Tokens kept by the chunk law (upper bound: K_c whole chunks)."""
    import math
    n_c = -(-w.N // w.chunk)
    ppm = int(math.floor(w.keep * 1e6 + 0.5))
    return max(1, min(n_c, (ppm * n_c + 999999) // 1000000)) * w.chunk


def resolve_shard(args, world: int) -> str | None:
    if world == 1:
        return None
    if args.shard != "auto":
        return args.shard
    return {"C2": "batch", "C3": "seq", "C4": "seq"}.get(args.config, "replica")


# ---------------------------------------------------------------- cpu baseline (oracle)
def cpu_baseline(w, n_layers: int):
    """The float64 oracle as it stands, on this host's cores, on a bounded
    sample: request 0, the first n_layers layers over all N tokens, plus the
    full selection.  Scaled to tokens/s of the whole workload geometry."""
    import numpy as np
    from threadpoolctl import threadpool_info

    from oracle import ref
    from spgen import gen
    Ls = min(n_layers, w.L)
    Q = ref.bf16_to_f64(np.stack([gen.gen_Q(w, 0, l) for l in range(Ls)]))
    Ks = [ref.bf16_to_f64(np.stack([gen.gen_K(w, 0, l, g) for g in range(w.Hkv)])) for l in range(Ls)]
    t0 = time.perf_counter()
    imp = ref.token_importance(Q, lambda l: Ks[l], w.scale, w.Rv)
    t1 = time.perf_counter()
    ref.select(imp, w.keep, w.pool_k, w.chunk)
    t2 = time.perf_counter()
    t_req = (t1 - t0) * (w.L / Ls) + (t2 - t1)          # one whole request
    threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    return {"value": w.N / t_req, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"request 0 of {w.name}: layers 0..{Ls - 1} of {w.L} over all {w.N} tokens "
                      f"(scaled x{w.L / Ls:g}) + full selection; {t2 - t0:.1f} s of CPU work",
            "host_cpus": os.cpu_count()}


def run_reference(args):
    """--impl reference: the oracle is the reference arm (no reference code
    exists for this paper).  Rank 0 only; other ranks exit without work.

    Each step is a bounded sample of the workload, timed as it runs: the
    float64 scoring of request 0's first `layers` layers over all N prompt
    tokens plus the full selection (the inputs are generated once, untimed).
    ms_per_step is that sample's measured time, so steps x ms_per_step is the
    arm's timed wall clock; value counts the prompt-token equivalent of the
    work done per step, N * layers / L tokens."""
    import numpy as np

    from oracle import ref
    from spgen import gen
    from threadpoolctl import threadpool_info
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload(args.config)
    layers = max(1, min(w.L, 2))
    Q = ref.bf16_to_f64(np.stack([gen.gen_Q(w, 0, l) for l in range(layers)]))
    Ks = [ref.bf16_to_f64(np.stack([gen.gen_K(w, 0, l, g) for g in range(w.Hkv)])) for l in range(layers)]
    times = []
    for s_ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        imp = ref.token_importance(Q, lambda l: Ks[l], w.scale, w.Rv)
        ref.select(imp, w.keep, w.pool_k, w.chunk)
        t1 = time.perf_counter()
        if s_ >= args.warmup:
            times.append(t1 - t0)
    ms = 1000.0 * statistics.mean(times)
    tok_equiv = w.N * layers / w.L
    val = tok_equiv / (ms / 1000.0)
    threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    sample = (f"request 0 of {w.name}: float64 scoring of layers 0..{layers - 1} of {w.L} over all {w.N} tokens "
              f"+ the full selection per step ({tok_equiv:g} prompt-token equivalents per step)")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} {w.name}" + secondary_label(), "B": w.B, "N": w.N, "L": w.L, "H": w.H,
                       "Hkv": w.Hkv, "d": w.d, "R": w.R, "keep": w.keep, "pool_k": w.pool_k, "chunk": w.chunk,
                       "sampled_layers": layers, "prompt_token_equiv_per_step": tok_equiv},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                             "host_cpus": os.cpu_count()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_2502_02789_b200 as sp
    from spgen import cuda as spgen_cuda

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workload(args.config)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    shard = resolve_shard(args, world)
    seq = shard in ("seq", "seq-split")
    seq_peer = shard == "seq"
    head = shard == "head"
    bsplit = shard == "batch"
    if shard == "replica":
        w = w.with_(seed=w.seed + rank)              # replicas: every rank its own copy of the workload
    if bsplit:
        from paper_2502_02789_b200 import dist as spd
        b0, b1 = spd.batch_range(w.B, world, rank)
        if b1 <= b0:
            raise SystemExit(f"--shard batch needs B >= world (B = {w.B})")

    # ---- inputs resident in HBM (device-side generator, bit-identical to spgen.gen)
    if seq:
        from paper_2502_02789_b200 import dist as spd
        i0, i1 = spd.token_range(w.N, world, rank)
        Q, K, T = spgen_cuda.make_inputs(w, device=dev, i0=i0, n_local=i1 - i0)
    else:
        Q, K, T = spgen_cuda.make_inputs(w, device=dev)
    if bsplit:                                       # this rank's requests [b0, b1) of the batch
        Q, K, T = Q[b0:b1].clone(), K[b0:b1].clone(), T[b0:b1].clone()
        w = w.with_(B=b1 - b0)
        torch.cuda.empty_cache()
    if head:                                         # this rank's heads (strided views of the whole inputs)
        from paper_2502_02789_b200 import dist as spd
        g0, g1 = spd.head_range(w.Hkv, world, rank)
        Qh_, Kh_ = Q[:, :, :, g0 * w.G:g1 * w.G], K[:, :, g0:g1]
        acc_buf = torch.empty((w.B, w.Rv, w.N), dtype=torch.float32, device=dev)
    f8 = args.kv == "e4m3"
    if f8:
        if seq or head:
            raise SystemExit("--kv e4m3 runs single-GPU or batch-sharded")
        from spgen import fp8
        Q8 = fp8.to_e4m3_codes(Q, fp8.Q_INV_SCALE)
        K8 = fp8.to_e4m3_codes(K, fp8.K_INV_SCALE)
        del K
        K = K8
    paged = args.paged > 0
    seq_lens, n_tokens = None, w.B * w.N
    if paged:
        if seq or head:
            raise SystemExit("--paged runs single-GPU or batch-sharded")
        from spgen.paged import to_paged
        K_cache, btab = to_paged(K, args.paged, seed=rank, layout=args.paged_layout)
        del K
        K = K_cache
        if args.ragged:
            import numpy as np
            lens = np.random.default_rng(1234 + rank).integers(w.N // 4, w.N + 1, size=w.B)
            lens[0] = w.N
            seq_lens = torch.tensor(lens, dtype=torch.int32, device=dev)
            n_tokens = int(lens.sum())
    torch.cuda.synchronize()
    imp = torch.empty((w.B, w.N), dtype=torch.float32, device=dev)
    ids = torch.empty((w.B, w.N), dtype=torch.int32, device=dev)
    pos = torch.empty_like(ids)
    nk = torch.empty((w.B,), dtype=torch.int32, device=dev)
    out = torch.empty_like(ids)

    def score_only():
        if paged and f8:
            sp.score_paged(Q8, K_cache, btab, seq_lens, N=w.N, R_valid=w.Rv, scale=w.scale, out=imp,
                           q_scale=1.0 / fp8.Q_INV_SCALE, k_scale=1.0 / fp8.K_INV_SCALE)
        elif paged:
            sp.score_paged(Q, K_cache, btab, seq_lens, N=w.N, R_valid=w.Rv, scale=w.scale, out=imp)
        elif f8:
            sp.score_e4m3(Q8, K8, 1.0 / fp8.Q_INV_SCALE, 1.0 / fp8.K_INV_SCALE, R_valid=w.Rv, scale=w.scale, out=imp)
        else:
            sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=imp, algo=args.algo)

    def select_only():
        if seq_lens is not None:
            sp.select_ragged(imp, seq_lens, w.keep, w.pool_k, w.chunk, w.pos0, tokens=T)
            return
        sp.select(imp, w.keep, w.pool_k, w.chunk, w.pos0, ids=ids, pos=pos, n_kept=nk, tokens=T, out=out)

    def step():
        score_only()
        select_only()

    # the plain single-GPU step goes through sp_score_select: the score kernel
    # without its cross-unit-group epilogue, the selection launch finalizing the
    # importance from the partial maps (same bits); --two-launch:
    # sp_score then sp_select_gather
    fused_step = not (args.two_launch or paged or f8 or args.algo == "simt" or seq_lens is not None)
    sel_out = {"importance": imp, "ids": ids, "pos": pos, "n_kept": nk, "out_tokens": out}
    if fused_step:
        def step():                                    # noqa: F811
            sp.score_select(Q, K, w.keep, w.pool_k, w.chunk, w.pos0, tokens=T, R_valid=w.Rv, scale=w.scale,
                            out=sel_out)

    peer_note = None

    def all_agree_failed(failed: bool) -> bool:        # a collective decision: any rank failed
        t = torch.tensor([1 if failed else 0], device=dev, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return bool(t.item())

    if seq_peer:
        from paper_2502_02789_b200 import dist as spd
        err = None
        try:
            peer_ptrs, peer_ws = spd._peer_buffers(Q, K, w.Rv, None)
        except Exception as e:                                      # noqa: BLE001
            err = e
        if all_agree_failed(err is not None):
            # the symmetric-memory peer exchange is not available here: the NCCL-only split
            seq_peer, shard = False, "seq-split"
            peer_note = f"peer exchange setup failed ({type(err).__name__ if err else 'on another rank'}): seq-split"
    if seq:
        from paper_2502_02789_b200 import dist as spd
        imp_loc = torch.empty((w.B, K.shape[3]), dtype=torch.float32, device=dev)

        def score_only():                              # noqa: F811 -- the sharded scoring (with its exchange)
            if seq_peer:                               # one pass: the exchange runs in the kernel, over NVLink
                sp.score_peer(Q, K, rank, world, peer_ptrs, 0, w.Rv, w.scale, out=imp_loc, ws=peer_ws)
                return
            st_ = sp.score_stats(Q, K, w.Rv, w.scale)
            parts = torch.empty((world * st_.shape[0], 2), dtype=torch.float32, device=dev)
            dist.all_gather_into_tensor(parts, st_)
            lse2 = sp.stats_combine(parts.view(world, -1, 2))
            sp.score_finish(Q, K, lse2, w.Rv, w.scale, out=imp_loc)

        def step():                                    # noqa: F811
            score_only()
            # the sharded selection: edges + candidate all-gathers, global merge (no importance all-gather)
            spd.seq_sharded_select(imp_loc, w.N, w.keep, w.pool_k, w.chunk, w.pos0, T)

    if head:
        def score_only():                              # noqa: F811 -- head-sharded scoring + MAX all-reduce
            sp.score_acc(Qh_, Kh_, w.Rv, w.scale, out=acc_buf)
            dist.all_reduce(acc_buf, op=dist.ReduceOp.MAX)
            sp.acc_importance(acc_buf, out=imp)

        def step():                                    # noqa: F811
            score_only()
            select_only()

    tuned = None
    if not (args.no_tune or args.plan or seq or head or paged or args.algo == "simt"):
        if f8:
            tuned = sp.score_e4m3_tune(Q8, K8, 1.0 / fp8.Q_INV_SCALE, 1.0 / fp8.K_INV_SCALE, w.Rv, w.scale)
        else:
            tuned = sp.score_tune(Q, K, w.Rv, w.scale)     # setup, not timed; later calls use the winner
    for _ in range(args.warmup):
        step()
    if seq_peer:
        # a peer exchange that cannot complete (e.g. peer memory not reachable) ends in
        # SP_ETIMEOUT: decided on every rank together, fall back to the NCCL-only split
        failed = False
        try:
            sp.check_device_error()
        except sp.SpError as e:                                     # noqa: BLE001
            failed, peer_note = True, f"peer exchange failed in warm-up ({e}): seq-split"
        if all_agree_failed(failed):
            seq_peer, shard = False, "seq-split"
            peer_note = peer_note or "peer exchange failed on another rank in warm-up: seq-split"
            for _ in range(args.warmup):
                step()
    sp.check_device_error()

    # CUDA graphs: the K timed steps captured as ONE graph (and the K score
    # launches of the roofline timing as another), so the device runs them back
    # to back with no per-step host launch gap; a one-step graph for warm-up
    graph_note = "eager"
    run_step, run_score = step, score_only
    run_steps = run_scores = None
    if not args.no_graph and not (seq or head):
        try:
            g_step, g_steps, g_scores = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_step):
                step()
            with torch.cuda.graph(g_steps):
                for _ in range(args.steps):
                    step()
            with torch.cuda.graph(g_scores):
                for _ in range(args.steps):
                    score_only()
            run_step = g_step.replay
            run_steps, run_scores = g_steps.replay, g_scores.replay
            for _ in range(2):
                run_step()
            run_steps()
            run_scores()
            torch.cuda.synchronize()
            sp.check_device_error()
            graph_note = "cuda-graph (the K timed steps replayed as one graph)"
        except Exception as e:                                   # noqa: BLE001
            graph_note = f"eager (graph capture failed: {type(e).__name__})"
            run_step, run_score = step, score_only
            run_steps = run_scores = None

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    if run_steps is not None:
        run_steps()
    else:
        for _ in range(args.steps):
            run_step()
    t_end.record(stream)
    barrier()
    # the dominant kernel alone, same launch configuration, same stream.  The
    # sequence-sharded peer kernel needs a cross-rank barrier between launches
    # (its rank-word buffers alternate halves): each launch is bracketed by its
    # own events and the barrier sits outside them.
    if seq_peer:
        score_ms = 0.0
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_score()
            e1.record(stream)
            barrier()
            score_ms += e0.elapsed_time(e1)
        score_ms /= args.steps
    else:
        s_start = torch.cuda.Event(enable_timing=True)
        s_end = torch.cuda.Event(enable_timing=True)
        s_start.record(stream)
        if run_scores is not None:
            run_scores()
        else:
            for _ in range(args.steps):
                run_score()
        s_end.record(stream)
        barrier()
    clk = clocks.stop()
    sp.check_device_error()
    ms_total = t_start.elapsed_time(t_end)
    if not seq_peer:
        score_ms = s_start.elapsed_time(s_end) / args.steps
    fused_ms = None
    if dist is not None:
        tt = torch.tensor([ms_total, score_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total, score_ms = tt.tolist()
    score_only_ms = score_ms
    if fused_ms is not None:
        score_ms = fused_ms
    ms_step = ms_total / args.steps
    # seq / head: every rank works on the same prompt (strong scaling); batch split and
    # replicas: the ranks' own requests add up (batch split: the one batch, strong)
    tokens_per_step = n_tokens
    if world > 1 and not (seq or head):
        tt = torch.tensor([n_tokens], device=dev, dtype=torch.int64)
        dist.all_reduce(tt)
        tokens_per_step = int(tt.item())
    value = tokens_per_step / (ms_step / 1000.0)

    # ---- roofline of the dominant kernel (sp_score): algorithmic bytes / duration
    peak, peak_src = peaks()
    esz = 1 if f8 else 2
    q_bytes = w.B * w.L * w.Rv * w.H * w.d * esz
    k_bytes = w.k_bytes // 2 * esz * n_tokens // (w.B * w.N)
    alg_bytes = ((k_bytes // world if (seq or head) else k_bytes) + (q_bytes // world if head else q_bytes)
                 + w.B * w.N * 4)
    achieved = alg_bytes / (score_ms / 1000.0) / 1e9
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and not (seq or head or bsplit):
        with open(tp) as f:
            tj = json.load(f)
        key = f"{args.config}/{args.algo}" + ("/e4m3" if f8 else "") + (f"/paged{args.paged}" if paged else "") \

        traffic = tj.get(key)
        traffic_src = tj.get("_source", {}).get(key) if traffic is not None else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "sp_score" + (" (timed alone, with its cross-unit-group epilogue; the step runs "
                                        "sp_score_select, where the selection launch does that finalize)"
                                        if fused_step else ""),
                "kernel_ms": score_ms, "score_only_ms": score_only_ms,
                "algorithmic_bytes": alg_bytes, "peak_source": peak_src,
                "frac_of_8TBs": achieved / SPEC_HBM_GBS, "score_share_of_step": score_ms / ms_step}

    # ---- end to end through the C ABI with host (pinned) buffers
    e2e = None
    if not args.no_e2e and not (seq or head or f8 or paged):    # sp_run_host is the single-GPU / batch-sharded bf16 call
        e2e = run_e2e(args, w, Q, K, T, dev, stream, dist, tokens_per_step)
    read_peak = None
    if not args.no_read_peak:
        from spgen import cuda as spgen_cuda2
        rp = spgen_cuda2.read_stream_gbs(dev)
        best = max(rp.values())
        read_peak = {"gbs": best, "frac": achieved / best, "probes_gbs": rp,
                     "how": "best of 10 passes over a 2 GiB buffer: 1-D TMA bulk copies into a 6-stage SMEM ring "
                            "(one CTA per SM) and 128-bit ld.global.nc read-xor (spgen/probe.cu), CUDA events"}
    roofline["read_peak"] = read_peak

    # select_gather is one launch (phase A over several CTAs for long prompts, the
    # last of them continuing with the top-K: launch_select() in csrc/select.cu)
    def sel_launches(n_tok):
        return 1
    if seq:
        n_loc = w.N // world
        sel = (1 if w.pool_k > 1 else 0) + sel_launches(n_loc) + 1         # edges, candidates, merge
        launches_per_step = (1 if seq_peer else 2 + 1) + sel                 # score_peer | stats+combine+finish
    elif fused_step:
        launches_per_step = 2                                 # score, dependent selection (finalize + select)
    else:
        launches_per_step = {"fused": 1, "simt": 4, "auto": 1}[args.algo] + sel_launches(w.N) \
            + (1 if head else 0)
    Kgeom = (torch.empty(w.d, dtype=torch.bfloat16, device=dev).as_strided((w.B, w.L, w.Hkv, w.N, w.d),
                                                                          (0, 0, 0, 0, 1)) if paged else K)
    Kgeom8 = (torch.empty(w.d, dtype=torch.uint8, device=dev).as_strided((w.B, w.L, w.Hkv, w.N, w.d),
                                                                        (0, 0, 0, 0, 1)) if paged and f8 else None)
    plan = ((sp.score_e4m3_plan(Q8, Kgeom8 if paged else K8, w.Rv) if f8 else sp.score_plan(Q, Kgeom, w.Rv))
            if args.algo != "simt" else None)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if (seq or head or bsplit) else "weak", "vs_baseline": None, "dtype": args.kv, "data": "synthetic",
            "config": {"workload": f"{args.config} {w.name}" + secondary_label() + (" e4m3 K/Q" if f8 else "")
                       + (f" paged bs{args.paged} {args.paged_layout}" if paged else "") + (" ragged" if seq_lens is not None else ""),
                       "prompt_tokens_per_step": n_tokens, "B": w.B, "N": w.N, "L": w.L, "H": w.H, "Hkv": w.Hkv,
                       "d": w.d, "R": w.R, "keep": w.keep, "pool_k": w.pool_k, "chunk": w.chunk,
                       "algo": args.algo, "plan": plan, "plan_tuned": tuned, "launch": graph_note, "shard": shard,
                       "shard_note": peer_note,
                       "parallelism": (f"seq{world} (prompt split, in-kernel statistics exchange over NVLink "
                                       f"peer memory, sharded select: candidate all-gather + merge)" if seq_peer else
                                       f"seq{world} (prompt split, NCCL stats all-gather, sharded select)" if seq else
                                       f"tp{world} (head split, NCCL MAX all-reduce of the log-domain maxima)"
                                       if head else
                                       f"dp{world} (batch split: requests [{b0}, {b1}) on rank {rank}, no collective)"
                                       if bsplit else
                                       f"replica{world} (every rank its own copy, no collective)")
                       if world > 1 else "single",
                       "l2": f"inputs larger than L2 (K = {k_bytes / 2**30:.2f} GiB per GPU), no flush"},
            "roofline": roofline, "clocks": clk, "e2e": e2e, "gpu_launches": launches_per_step * args.steps}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_sample_layers)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_e2e(args, w, Q, K, T, dev, stream, dist, job_tokens):
    """Same metric through sp_run_host: H2D of the step's inputs from pinned
    host memory, score/select/gather, D2H of ids/pos/n_kept/tokens."""
    import torch

    import paper_2502_02789_b200 as sp
    Qh = Q.cpu().pin_memory()
    Kh = K.cpu().pin_memory()
    Th = T.cpu().pin_memory()
    ho = {k: torch.empty((w.B, w.N), dtype=torch.int32).pin_memory() for k in ("ids", "pos", "out_tokens")}
    ho["n_kept"] = torch.empty((w.B,), dtype=torch.int32).pin_memory()
    nbytes = sp.run_workspace_bytes(Q, K, w.keep, w.pool_k, w.chunk, w.Rv, w.scale, w.pos0)
    dv = {"Q": torch.empty_like(Q), "K": torch.empty_like(K), "tokens": torch.empty_like(T),
          "importance": torch.empty((w.B, w.N), dtype=torch.float32, device=dev),
          "ids": torch.empty_like(T), "pos": torch.empty_like(T), "n_kept": torch.empty((w.B,), dtype=torch.int32,
                                                                                      device=dev),
          "out_tokens": torch.empty_like(T), "ws": torch.zeros(nbytes, dtype=torch.uint8, device=dev)}
    steps = max(2, min(args.steps, 5))
    for _ in range(2):
        sp.run_host(Qh, Kh, Th, dv, w.keep, w.pool_k, w.chunk, w.Rv, w.scale, w.pos0, host_out=ho)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        sp.run_host(Qh, Kh, Th, dv, w.keep, w.pool_k, w.chunk, w.Rv, w.scale, w.pos0, host_out=ho)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    h2d = Qh.numel() * 2 + Kh.numel() * 2 + Th.numel() * 4
    d2h = 3 * w.B * w.N * 4 + w.B * 4
    return {"value": job_tokens / (ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": steps}


def main():
    args = parse()
    _SECONDARY.update(R=args.R, chunk=args.chunk, pool_k=args.pool, keep=args.keep)
    if args.plan:
        os.environ["SP_FUSED_PLAN"] = args.plan
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
