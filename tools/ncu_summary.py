"""Summarise the ncu evidence of one gpurun call into profiles/ (tracked).

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launch_list_summary.txt
  python tools/ncu_summary.py full gpurun_out/pass_full.ncu-rep profiles/r01_ncu_update_kernels.json

`launches`: the `--metrics gpu__time_duration.sum --clock-control none` launch list
(per-launch times are cold-cache and serialised: compare shares).  `full`: the
headline pipe / DRAM / stall metrics of each kernel in an `ncu --set full` report.
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    "gpu__time_duration.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__inst_executed.sum.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size",
    "launch__block_size",
]


def launches(src, dst, cmd=""):
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    head = rows[0]
    ki, vi, mi = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Name")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + float(r[vi].replace(",", "")))
    tot = sum(t for _, t in agg.values())
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none -- %s" % cmd,
           "units: ms; per-launch times are cold-cache and serialised: compare SHARES",
           "kernel, launches, total_ms, mean_ms, share"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append("%s, %d, %.3f, %.4f, %.4f" % (name, n, t * 1e-6, t * 1e-6 / n, t / tot))
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:12]))


def full(src, dst, note=""):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], stdout=subprocess.PIPE,
                         stderr=subprocess.DEVNULL, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    res = OrderedDict(source=note or src)
    for r in rows[2:]:
        name = r[head.index("Kernel Name")]
        d = OrderedDict()
        for m in FULL_METRICS:
            if m in head:
                d[m] = r[head.index(m)]
        d["units"] = {m: units[head.index(m)] for m in FULL_METRICS if m in head}
        stalls = {}
        for i, h in enumerate(head):
            p = "smsp__average_warps_issue_stalled_"
            if h.startswith(p) and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len(p):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        d["stalls_per_issue"] = OrderedDict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
        key = name
        k = 2
        while key in res:
            key = "%s #%d" % (name, k)
            k += 1
        res[key] = d
    json.dump(res, open(dst, "w"), indent=1)
    for k, v in res.items():
        if isinstance(v, dict):
            print(k, {m: v.get(m) for m in FULL_METRICS[:6]})


if __name__ == "__main__":
    what, src, dst = sys.argv[1:4]
    extra = " ".join(sys.argv[4:])
    launches(src, dst, extra) if what == "launches" else full(src, dst, extra)
