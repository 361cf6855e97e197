#!/bin/bash
# ncu --set full of the HBM-bound kernels of one cfg5 step (after warm-up)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_predict|k_resample_gather|k_scan_chunks|k_records" --launch-skip 12 -c 4 -f -o gpurun_out/hbm_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_hbm.log 2>&1; echo ncu_hbm=$?
