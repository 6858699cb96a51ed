"""Write a markdown summary of an ncu --set full report (+ launch list, + bench JSON)
into profiles/, and the per-launch DRAM traffic of the Ax kernel into
profiles/traffic.json (read by bench.py for roofline.traffic).

  python tools/summarize_profile.py <report.ncu-rep> <launches.csv> <bench.json-line file> <tag>
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def raw(reps):
    h = units = None
    rows = []
    for rep in reps.split(","):
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rr = list(csv.reader(out.splitlines()))
        if h is None:
            h, units = rr[0], rr[1]
        idx = [rr[0].index(c) if c in rr[0] else None for c in h]
        for r in rr[2:]:
            rows.append([r[i] if i is not None else "" for i in idx])
    return h, units, rows


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    t = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            t.setdefault(r[ki].split("(")[0][:60], []).append(float(r[vi].replace(",", "")) / 1e3)
    return t


def main():
    rep, lcsv, bench, tag = sys.argv[1:5]
    h, units, rows = raw(rep)
    ki = h.index("Kernel Name")
    lines = [f"# Profile summary {tag}", "",
             "ncu --set full --clock-control none (cold cache per replay, serialised); "
             "source: `" + rep + "`", "",
             "| kernel | " + " | ".join(m[1] for m in METRICS) + " |",
             "|---" * (len(METRICS) + 1) + "|"]
    seen = OrderedDict()
    for r in rows:
        name = r[ki].split("(")[0]
        if name.startswith("void "):
            name = name[5:]
        if name in seen:
            continue
        seen[name] = r
        vals = []
        for m, _ in METRICS:
            v = r[h.index(m)] if m in h else ""
            u = units[h.index(m)] if m in h else ""
            vals.append(f"{v} {u}".strip())
        lines.append(f"| `{name}` | " + " | ".join(vals) + " |")
    lines += ["", "## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
              "| kernel | launches | mean us | total us |", "|---|---|---|---|"]
    tot_all = 0.0
    lt = launches(lcsv)
    for k, v in lt.items():
        tot_all += sum(v)
    for k, v in lt.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} |")
    if os.path.exists(bench):
        d = json.loads(open(bench).read().strip().splitlines()[-1])
        lines += ["", "## bench.py line (same code)", "", "```json", json.dumps(d, indent=1), "```"]
    out = os.path.join(ROOT, "profiles", f"{tag}_summary.md")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    open(out, "w").write("\n".join(lines) + "\n")
    # traffic of the PCG Ax kernel (AX_PCG = mode 2, n = 8)
    traffic = {}
    # prefer the one-rank PCG kernel with the fused p update (<8, 2, 0, 1>)
    cands = [r for name, r in seen.items() if "ax_kernel" in name and "<8, 2" in r[ki]]
    cands.sort(key=lambda r: 0 if ("<8, 2, 0, 1>" in r[ki] or "true>" in r[ki]) else 1)
    for r in cands[:1]:
        full = r[ki]
        b = float(r[h.index("dram__bytes_read.sum")]) + float(r[h.index("dram__bytes_write.sum")])
        scale = 1e6 if units[h.index("dram__bytes_read.sum")].lower().startswith("m") else 1.0
        traffic["C2_N7_P1"] = {"kernel": full[:80], "dram_bytes_per_launch": b * scale,
                               "source": os.path.basename(rep)}
    if traffic:
        json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
