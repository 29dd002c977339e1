"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` log into a
per-kernel launch table (total ms, share, launch count):
    python tools/launch_table.py LOG OUT.txt "command line"
"""
import collections
import csv
import sys

log, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(l for l in open(log) if l.startswith('"')))
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tot = collections.defaultdict(float)
cnt = collections.Counter()
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "s": 1e3, "second": 1e3}
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    cnt[name] += 1
T = sum(tot.values())
lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none: {cmd}",
         "# (cold-cache, serialised launches; shares, not absolute step times)",
         f"# total kernel time {T / 1e3:.3f} s over {sum(cnt.values())} launches"]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    lines.append(f"{v:14.4f} ms {100 * v / T:8.3f}% x{cnt[k]:<5d} {k[:110]}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:14]))
