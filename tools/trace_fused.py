"""Timeline of the fused score kernel from its globaltimer trace (debug tool).

  python tools/trace_fused.py [--config C3] [--plan n_tg,n_ug]

Event ids per (CTA, unit): 0 producer starts unit, 1 MMA starts (slot free),
2 stats start, 3 CTA partial published, 4 partials cleanup done, 5 lse2 ready
(this CTA combined all partials), 6 aggregation done, 7 stats compute done.
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--plan", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--kv", default="bf16", choices=["bf16", "e4m3"])
    a = ap.parse_args()
    if a.plan:
        os.environ["SP_FUSED_PLAN"] = a.plan
    w = gen.CONFIGS[a.config]
    Q, K, T = spgen_cuda.make_inputs(w)
    if a.kv == "e4m3":
        from spgen import fp8
        Q8, K8 = fp8.to_e4m3_codes(Q, fp8.Q_INV_SCALE), fp8.to_e4m3_codes(K, fp8.K_INV_SCALE)
        plan = sp.score_e4m3_plan(Q8, K8, w.Rv)

        def run():
            sp.score_e4m3(Q8, K8, 1 / fp8.Q_INV_SCALE, 1 / fp8.K_INV_SCALE, R_valid=w.Rv, scale=w.scale)
    else:
        plan = sp.score_plan(Q, K, w.Rv)

        def run():
            sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    grid, upj = plan["grid"], plan["units_per_job"]
    units = upj * ((w.B * plan["jobs_per_request"] + grid - 1) // grid)
    buf = torch.zeros(grid * (units + 1) * 8 + 1000 * 8, dtype=torch.int64, device="cuda")   # +1: wait accounting; CTA 0 tiles
    for _ in range(3):
        run()
    sp.lib().sp_trace_enable(buf.data_ptr(), buf.numel())
    run()
    torch.cuda.synchronize()
    sp.lib().sp_trace_enable(None, 0)
    tt = buf[grid * (units + 1) * 8:].view(1000, 8).cpu().numpy().astype(np.float64)
    full = buf[:grid * (units + 1) * 8].view(grid, units + 1, 8).cpu().numpy().astype(np.float64)
    waits = full[:, units, :7] / 1965.0                          # SM cycles -> us (1965 MHz)
    tr = full[:, :units, :]
    t0 = tr[tr > 0].min()
    tr = np.where(tr > 0, (tr - t0) / 1000.0, np.nan)            # microseconds from the first stamp
    if a.out:
        np.save(a.out, tr)
    print("plan", plan, "units/CTA", units)
    n = int((tt[:, 3] > 0).sum())
    if n > 1:
        t = tt[:n, :4] - tt[0, 0]
        print("CTA 0 MMA per tile (cycles): wait slot / wait full / issue ; period")
        for i in list(range(0, 24)) + list(range(n // 2, n // 2 + 16)):
            if i < n:
                print("  tile %4d  slot %6.0f  full %6.0f  issue %6.0f  period %6.0f" % (
                    i, t[i, 1] - t[i, 0], t[i, 2] - t[i, 1], t[i, 3] - t[i, 2], (t[i, 0] - t[i - 1, 0]) if i else 0))
        print("  globaltimer ns per tile (period): %.1f ; issue ns mean %.1f" % (np.mean(np.diff(tt[:n, 4])), np.mean(tt[:n, 5] - tt[:n, 4])))
        print("  mean: slot %.0f full %.0f issue %.0f period %.0f" % (np.mean(t[:, 1] - t[:, 0]), np.mean(t[:, 2] - t[:, 1]),
              np.mean(t[:, 3] - t[:, 2]), np.mean(np.diff(t[:, 0]))))
    print("kernel span (us) %.1f" % np.nanmax(tr))
    wn = ["prod wait empty", "prod wait qempty", "mma wait qfull", "mma wait tmem slot", "mma wait tma full",
          "mma span", "mma issue+commit"]
    for k, nm in enumerate(wn):
        print(f"{nm:>20}: mean {waits[:, k].mean():8.1f} us  min {waits[:, k].min():8.1f}  max {waits[:, k].max():8.1f}")
    names = ["prod", "mma", "stats", "publ", "cleanup", "lseready", "aggdone", "statsend"]
    for (x, y) in [(1, 2), (2, 7), (7, 3), (3, 5), (5, 6), (1, 6), (0, 1)]:
        d = tr[:, :, y] - tr[:, :, x]
        print(f"{names[x]:>8} -> {names[y]:<8} mean {np.nanmean(d):8.2f} us  p50 {np.nanmedian(d):8.2f}  max {np.nanmax(d):8.2f}")
    # per-unit period: successive MMA starts
    per = np.diff(tr[:, :, 1], axis=1)
    print("MMA start period per unit: mean %.2f us  p50 %.2f" % (np.nanmean(per), np.nanmedian(per)))
    per = np.diff(tr[:, :, 6], axis=1)
    print("agg done period per unit:  mean %.2f us  p50 %.2f" % (np.nanmean(per), np.nanmedian(per)))
    # skew: for each unit index, spread of publish times across CTAs
    pub = tr[:, :, 3]
    print("publish skew across CTAs per unit (max-min): mean %.2f us" % np.nanmean(np.nanmax(pub, 0) - np.nanmin(pub, 0)))
    # lateness of each CTA vs the median publish time of the CTAs sharing its units
    n_tg, n_ug = plan["token_groups"], plan["unit_groups"]
    late = np.full(grid, np.nan)
    if w.B * plan["jobs_per_request"] <= grid:
        for ug in range(n_ug):
            ctas = [tg * n_ug + ug for tg in range(n_tg) if tg * n_ug + ug < grid]
            med = np.nanmedian(pub[ctas], axis=0)
            for c in ctas:
                late[c] = np.nanmean(pub[c] - med)
        order = np.argsort(-np.nan_to_num(late, nan=-1e9))
        print("CTA lateness vs median publish (us): mean %.2f  p90 %.2f  max %.2f" % (
            np.nanmean(late), np.nanpercentile(late, 90), np.nanmax(late)))
        print("  latest CTAs:", ", ".join("%d(%.1f)" % (c, late[c]) for c in order[:12]))
        # late CTA's own lag: when did it start each unit's stats relative to others
        st = tr[:, :, 2]
        print("  stats-start lateness of latest CTA per unit (first 10 units):",
              " ".join("%.1f" % (st[order[0], u] - np.nanmedian(st[:, u])) for u in range(min(10, units))))
        print("  end time per CTA (agg done last unit): min %.1f  median %.1f  max %.1f" % (
            np.nanmin(tr[:, -1, 6]), np.nanmedian(tr[:, -1, 6]), np.nanmax(tr[:, -1, 6])))
    for c in [0, grid // 2, grid - 1]:
        print(f"CTA {c}: first units (us):")
        for u in range(min(4, units)):
            print("   ", " ".join(f"{x:8.1f}" for x in tr[c, u, :7]))


if __name__ == "__main__":
    main()
