"""Summarise ncu artefacts into profiles/ (tracked).

  python tools/ncu_summary.py <round-tag> <launches.csv> <report.ncu-rep>...

Writes profiles/<tag>_launches.md (per-kernel launch list: count, mean device
time, share of the listed launches), profiles/<tag>_<kernel>.md (key metrics of
one --set full capture) and merges dram traffic per launch into
profiles/traffic.json (read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__bytes.min.per_second", "DRAM partition min BW"),
    ("dram__bytes.max.per_second", "DRAM partition max BW"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "TMEM/tensor memory active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic SMEM/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions executed"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    return [{h[i]: (r[i], u[i]) for i in range(len(h))} for r in rows[2:]]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    tag, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    os.makedirs(PROF, exist_ok=True)
    # ---- launch list
    rows = [r for r in csv.reader(l for l in open(launches) if not l.startswith("=="))]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
    def is_step(k):          # kernels of the timed step (input generation / torch fills are setup)
        return k.startswith("sp::")
    tot = sum(sum(v) for k, v in agg.items() if is_step(k))
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write(f"# {tag}: launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)\n\n")
        f.write("Cold-cache, serialised per-launch device times: compare shares, not absolutes.\n\n")
        f.write("| kernel | launches | mean time (us) | share of the step |\n|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda kv: (not is_step(kv[0]), -sum(kv[1]))):
            share = f"{sum(v) / tot * 100:.1f}%" if is_step(k) else "setup (input generation)"
            f.write(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1000:.1f} | {share} |\n")
    # ---- full captures
    tp = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    for rep in reps:
        for d in raw(rep):
            name = d["Kernel Name"][0].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
            lines = [f"# {tag}: `{d['Kernel Name'][0][:120]}`\n", f"source: `{os.path.basename(rep)}` (ncu --set full)\n\n",
                     "| metric | value | unit |\n|---|---|---|\n"]
            for key, label in KEYS:
                if key in d:
                    lines.append(f"| {label} (`{key}`) | {d[key][0]} | {d[key][1]} |\n")
            if "dram__bytes_read.sum" in d:
                t = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
                lines.append(f"\nDRAM traffic per launch (read+write): {t:.6g} bytes\n")
                cfg = os.environ.get("TRAFFIC_KEY")
                if cfg and name == os.environ.get("TRAFFIC_KERNEL", name):
                    traffic[cfg] = t
            with open(os.path.join(PROF, f"{tag}_{name}.md"), "w") as f:
                f.writelines(lines)
    with open(tp, "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main()
