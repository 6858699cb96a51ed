"""Top SASS lines by warp-stall samples for kernels in an ncu report (source page)."""
import csv
import subprocess
import sys

rep, flt = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
sections, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = {"name": ln, "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(ln)
for s in sections:
    if flt not in s["name"]:
        continue
    rows = list(csv.reader(s["rows"]))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    ii = h.index("Instructions Executed")
    data = [(int(r[si] or 0), r[1].strip(), r[ii]) for r in rows[1:] if len(r) > si]
    tot = sum(d[0] for d in data)
    print(s["name"][:120], "total samples", tot, "instructions", sum(int(d[2] or 0) for d in data))
    for smp, src, ex in sorted(data, reverse=True)[:top]:
        print(f"{smp:7d} {100.0 * smp / max(tot, 1):5.1f}%  {ex:>9s}  {src}")
    break
