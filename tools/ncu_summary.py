"""Summarise ncu captures into profiles/ (markdown + traffic.json for bench.py).

Usage: python tools/ncu_summary.py <round-tag> <name>=<report.ncu-rep> ... [--launches csv]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__warps_active.avg.per_cycle_active", "warps active / SMSP"),
    ("smsp__warps_eligible.avg.per_cycle_active", "warps eligible / SMSP"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
    stalls = []
    for h, (v, u) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    return d, sorted(stalls, reverse=True)[:6]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    seen_step = False  # launches before the first K1 are the one-time load (registration)
    for r in data:
        name = r[ik].split("(")[0].split("<")[0].split("::")[-1]
        seen_step = seen_step or name.startswith("prefix_attn")
        if not seen_step:
            name += " (load, one-time)"
        v = float(r[iv].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1e-3)
        agg[name].append(v * scale)
    return agg


def main():
    tag = sys.argv[1]
    reps = [a.split("=", 1) for a in sys.argv[2:] if "=" in a and not a.startswith("--")]
    lcsv = sys.argv[sys.argv.index("--launches") + 1] if "--launches" in sys.argv else None
    md = [f"# ncu summary — {tag}\n",
          "Captured on one B200 with `ncu --set full --clock-control none --import-source on` "
          "(cold-cache, serialised replays: compare shares and counters, not absolute times) "
          "on `python bench.py --profile --steps 2 --warmup 3` (C1 workload).\n"]
    traffic = {}
    for name, rep in reps:
        d, stalls = raw(rep)
        md.append(f"\n## {name}\n\n| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in d:
                v, u = d[key]
                md.append(f"| {label} (`{key}`) | {v} {u} |")
        md.append("\nTop stall reasons (warps per issue): " + ", ".join(f"{s} {v:.2f}" for v, s in stalls))
        def num(k):
            v, u = d.get(k, ("0", ""))
            x = float(v.replace(",", ""))
            return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
        traffic[name] = {"dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
                         "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
                         "report": os.path.basename(rep), "round": tag}
    if lcsv:
        agg = launches(lcsv)
        tot = sum(sum(v) for k, v in agg.items() if "one-time" not in k)  # share of the steps
        md.append("\n## launch list (`ncu --metrics gpu__time_duration.sum`)\n\nShare = of the decode steps' "
                  "kernel time (the one-time load launches are listed, not counted).\n\n"
                  "| kernel | launches | mean us | share |\n|---|---|---|---|")
        for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            share = "-" if "one-time" in n else f"{100*sum(v)/tot:.1f}%"
            md.append(f"| {n} | {len(v)} | {sum(v)/len(v):.2f} | {share} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w").write("\n".join(md) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    old = json.load(open(tp)) if os.path.exists(tp) else {}
    old.update(traffic)
    json.dump(old, open(tp, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
