#!/bin/bash
# round evidence (one gpurun call): GPU tests, default bench (dense line + gated leg), cfg3/cfg4 lines, launch lists, ncu --set full of the passes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu_tests=$?
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench=$?
for c in cfg3 cfg4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate.csv python bench.py --gate 1 --no-gated-leg --no-cpu-baseline > gpurun_out/ncu_gate.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass --launch-skip 6 -c 2 -o gpurun_out/pass_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_full.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gpass|k_psort_scatter" --launch-skip 9 -c 3 -o gpurun_out/gpass_full python bench.py --gate 1 --steps 1 --warmup 3 --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_gfull.log 2>&1; echo ncu4=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_predict|k_resample_mark|k_gather" --launch-skip 9 -c 3 -o gpurun_out/hbm_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_hbm.log 2>&1; echo ncu5=$?
timeout 900 python tools/table1_study.py --runs 10 --out gpurun_out/r01_table1_study > gpurun_out/table1.log 2>&1; echo table1=$?
