"""Plan sweep of the fused score kernel in one process (dev tool): for each
config and plan (n_tg, n_ug, hier) forced through SP_FUSED_PLAN, the mean
launch time over 20 launches (CUDA events), the HBM rate, and the importance's
max relative difference to the first plan's (all plans compute the same values
up to fp32 merge order).

  python tools/plan_sweep.py C3 37,4,0 37,4,1 64,2,1 [--kv e4m3] [C1 ...]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402


def sweep(name, plans, kv="bf16"):
    w = gen.CONFIGS[name]
    Q, K, T = spgen_cuda.make_inputs(w)
    f8 = kv == "e4m3"
    if f8:
        from spgen import fp8
        Q, K = fp8.to_e4m3_codes(Q, fp8.Q_INV_SCALE), fp8.to_e4m3_codes(K, fp8.K_INV_SCALE)
        qs, ks = 1.0 / fp8.Q_INV_SCALE, 1.0 / fp8.K_INV_SCALE
    out = torch.empty((w.B, w.N), dtype=torch.float32, device="cuda")
    ref = None
    kbytes = w.k_bytes // (2 if f8 else 1)

    def run():
        if f8:
            sp.score_e4m3(Q, K, qs, ks, R_valid=w.Rv, scale=w.scale, out=out)
        else:
            sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=out, algo="fused")

    for pl in plans:
        tg, ug, h = (int(x) for x in pl.split(","))
        os.environ["SP_FUSED_PLAN"] = pl
        got = sp.score_e4m3_plan(Q, K, w.Rv) if f8 else sp.score_plan(Q, K, w.Rv)
        if (got["token_groups"], got["unit_groups"], got["hier"]) != (tg, ug, h):
            print(f"{name} {kv} plan {pl}: invalid (got {got['token_groups']},{got['unit_groups']},{got['hier']})")
            continue
        for _ in range(4):
            run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()                     # 20 launches in one graph: no host overhead
        with torch.cuda.graph(g):
            for _ in range(20):
                run()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        sp.check_device_error()
        ms = a.elapsed_time(b) / 20
        if ref is None:
            ref = out.clone()
        err = ((out - ref).abs() / ref.abs().clamp_min(1e-30)).max().item()
        print(f"{name} {kv} plan {pl}: {ms:.4f} ms  {kbytes / ms / 1e6:.0f} GB/s  stages {got['stages']}  "
              f"rel diff {err:.1e}", flush=True)
    os.environ.pop("SP_FUSED_PLAN", None)
    del Q, K, T
    torch.cuda.empty_cache()


if __name__ == "__main__":
    args = sys.argv[1:]
    kv = "bf16"
    if "--kv" in args:
        i = args.index("--kv")
        kv = args[i + 1]
        del args[i:i + 2]
    cur, plans = None, []
    for a in args + ["END"]:
        if a in gen.CONFIGS or a == "END":
            if cur:
                sweep(cur, plans, kv)
            cur, plans = a, []
        else:
            plans.append(a)
