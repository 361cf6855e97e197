#!/bin/bash
# round-2 evidence (one gpurun call): GPU tests (near-tie log), bench cfg5 (default line incl.
# gated leg and CPU baseline), cfg4 (with its CPU baseline), cfg3, launch lists, ncu --set full
# of the dense passes (cfg5, cfg4) and of the HBM kernels
mkdir -p gpurun_out
export PHD_NEAR_TIE_LOG=gpurun_out/near_ties.json
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu_tests=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench5=$?
python bench.py --config cfg4 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4=$?
python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo bench3=$?
python bench.py --config cfg2 --no-cpu-baseline --no-gated-leg > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench2=$?
for c in cfg3 cfg2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_$c.log 2>&1; echo ncu_$c=$?
python tools/dbg/host_vs_gpu.py $c > gpurun_out/host_vs_gpu_$c.json 2>/dev/null; echo hvg_$c=$?
done
python tools/dbg/timeline.py cfg2 > gpurun_out/tl_cfg2.txt 2>&1; echo tl=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate.csv python bench.py --gate 1 --no-gated-leg --no-cpu-baseline > gpurun_out/ncu_gate.log 2>&1; echo ncu2=$?
CFGS="cfg5 cfg4" bash tools/gpu_ncu_passes.sh
bash tools/gpu_ncu_hbm.sh
