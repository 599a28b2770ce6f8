import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running full-size check")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Parity report: importance error and selection regime of every full-size case."""
    from tests import _util
    recs = _util.RECORDS
    if not recs:
        return
    import json
    n_exact = sum(r["regime"] == "exact" for r in recs)
    tr = terminalreporter
    tr.write_sep("-", f"parity report: {len(recs)} (config, seed, keep) cases, {n_exact} exact-regime, "
                      f"{len(recs) - n_exact} near-tie")
    for r in recs:
        m = "inf" if r["margin"] is None else f"{r['margin']:.3g}"
        tr.write_line(f"{r['where']:<28} {r['config']:<9} N={r['N']:<6} seed={r['seed']} {r['values']:<6} "
                      f"planted={int(r['planted'])} b={r['request']:<2} keep={r['keep']:<4} {r['regime']:<8} "
                      f"margin={m:<9} max_rel_err={r['max_rel_err']:.2e}")
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "parity_regimes.json"), "w") as f:
            json.dump(recs, f, indent=1)
