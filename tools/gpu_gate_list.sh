#!/bin/bash
# gated cfg5 (and cfg4) step: bench line + per-kernel launch list
mkdir -p gpurun_out
for c in ${CFGS:-cfg5}; do
python bench.py --config $c --gate 1 --no-gated-leg --no-cpu-baseline > gpurun_out/bench_gate_$c.json 2> gpurun_out/bench_gate_$c.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate_$c.csv python bench.py --config $c --gate 1 --no-gated-leg --no-cpu-baseline --steps 3 > gpurun_out/ncu_gate_$c.log 2>&1; echo ncu=$?
done
