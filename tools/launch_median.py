"""Per-kernel median launch time (us) of an ncu gpu__time_duration launch list.
  python tools/launch_median.py gpurun_out/launches_cfg3.csv"""
import csv
import statistics
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
t = defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    u = r[ui].strip()
    v = v / 1000.0 if u in ("nsecond", "ns") else (v * 1000.0 if u in ("msecond", "ms") else v)
    t[r[ki].split("(")[0][:60]].append(v)
for k, v in sorted(t.items(), key=lambda kv: -statistics.median(kv[1]) * len(kv[1])):
    print("%-60s n=%4d median %8.2f us" % (k, len(v), statistics.median(v)))
