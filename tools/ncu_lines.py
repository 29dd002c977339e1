"""Per-CUDA-source-line samples/instructions from an ncu report
(python tools/ncu_lines.py REP [N])."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname, hdr, cur = "", None, None
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:90])
    if cur is None:
        continue
    try:
        s = float(r[hdr["# Samples"]] or 0)
        ins = float(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, KeyError):
        continue
    a = agg[cur[:2]]
    a[0] += s
    a[1] += ins
    a[2] = cur[2]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts:.0f}, instructions {ti:.3e}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{k[0]}:{k[1]:<5} samp {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}% | {v[2]}")
