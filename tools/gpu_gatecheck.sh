#!/bin/bash
# gated-path check: gated + bounds tests, gated bench at cfg4 and cfg5, cfg4 gated launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gate.py tests/test_gpu_debug_bounds.py -x -q > gpurun_out/pytest_gate.log 2>&1; echo tests=$?
for c in cfg5 cfg4; do python bench.py --config $c --gate 1 --no-gated-leg --no-cpu-baseline > gpurun_out/bg_$c.json 2> gpurun_out/bg_$c.err; python -c "import json;d=json.load(open('gpurun_out/bg_$c.json'));print('$c',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms'].items()})"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_g4.csv python bench.py --config cfg4 --gate 1 --no-gated-leg --no-cpu-baseline --steps 3 > gpurun_out/ncu_g4.log 2>&1; echo ncu=$?
