#!/bin/bash
mkdir -p gpurun_out
for c in cfg1 cfg2; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --config cfg2 --no-cpu-baseline --no-gated-leg --steps 3 > gpurun_out/ncu_cfg2.log 2>&1; echo ncu=$?
