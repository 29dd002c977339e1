"""Print kernel/metric/value rows of an `ncu --csv --metrics ...` log.
    python tools/ncu_csv.py LOG [LOG ...]"""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    if not rows:
        print(path, "(no rows)")
        continue
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    for r in rows[1:]:
        print(path.split("/")[-1], r[ki][:40], r[mi], r[vi])
