"""Per-source-line warp-stall summary from an ncu report (needs -lineinfo).

  python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [file_substring] [N]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["long_sb", "no_inst", "sleep", "wait", "barrier", "selected", "short_sb", "math", "not_selected", "mio",
        "lg", "branch_resolving", "dispatch", "membar"]


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else "score_fused.cu"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, cols, cur_line = None, None, None
    by = collections.defaultdict(collections.Counter)
    src = {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1]
            continue
        if r[0] == "Line No":
            cols = {}
            for i, n in enumerate(r):
                cols.setdefault(n, i)
            continue
        if cols is None or cur_file is None or want not in cur_file:
            continue
        if r[0]:
            try:
                cur_line = int(r[0])
            except ValueError:
                continue
            src[cur_line] = r[1][:90]
        try:
            s = int(r[cols["Warp Stall Sampling (All Samples)"]])
        except (ValueError, IndexError, KeyError):
            continue
        c = by[cur_line]
        c["all"] += s
        for k in KEYS:
            try:
                c[k] += int(r[cols["stall_" + k]])
            except (ValueError, IndexError, KeyError):
                pass
    tot = collections.Counter()
    for c in by.values():
        tot.update(c)
    print("total samples", tot["all"], "|", ", ".join(f"{k}={tot[k]}" for k in sorted(KEYS, key=lambda k: -tot[k])))
    for ln, c in sorted(by.items(), key=lambda x: -x[1]["all"])[:top]:
        t = ", ".join(f"{k}={c[k]}" for k in sorted(KEYS, key=lambda k: -c[k])[:3] if c[k])
        print(f"{ln:5d} {c['all']:6d} | {t:48s} | {src.get(ln, '')}")


if __name__ == "__main__":
    main()
