#!/bin/bash
# per-kernel launch lists (ncu gpu__time_duration) of the small configs
mkdir -p gpurun_out
for c in ${CFGS:-cfg3 cfg2}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_$c.log 2>&1; echo ncu_$c=$?
python bench.py --config $c --no-cpu-baseline --no-gated-leg > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo bench_$c=$?
done
