#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"psort_scatter|k_gpass|k_ms_hist" --launch-skip 12 -c 4 -o gpurun_out/scatter_full python bench.py --gate 1 --no-gated-leg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sfull.log 2>&1; echo ncu2=$?
