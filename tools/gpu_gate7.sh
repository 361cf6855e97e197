#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu_tests=$?
timeout 600 python bench.py --gate 1 --no-gated-leg --no-cpu-baseline > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate.csv python bench.py --gate 1 --no-gated-leg --steps 3 --no-cpu-baseline > gpurun_out/ncu_gate.log 2>&1; echo ncu=$?
