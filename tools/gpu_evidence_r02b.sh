#!/bin/bash
# round-2 refresh after the late gated changes (one gpurun call): GPU tests, bench cfg5 / cfg4 /
# cfg3 (cfg5 and cfg4 with their CPU baselines and gated legs), gated launch lists (exact,
# gate_floor), the gated step's CUPTI timeline
mkdir -p gpurun_out
export PHD_NEAR_TIE_LOG=gpurun_out/near_ties.json
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu_tests=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench5=$?
python bench.py --config cfg4 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4=$?
python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo bench3=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate.csv python bench.py --gate 1 --no-gated-leg --no-cpu-baseline > gpurun_out/ncu_gate.log 2>&1; echo ncu2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate_floor.csv python bench.py --gate 1 --gate-floor -71 --no-gated-leg --no-cpu-baseline > gpurun_out/ncu_gate_floor.log 2>&1; echo ncu3=$?
GATE=1 NPROF=2 python tools/dbg/timeline.py cfg5 > gpurun_out/tl_gate_cfg5.txt 2>&1; echo tl=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gpass|k_psort_scatter" --launch-skip 6 -c 3 -f -o gpurun_out/gpass_full python bench.py --gate 1 --no-gated-leg --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_gpass.log 2>&1; echo ncu_gpass=$?
python tools/ncu_summary.py full gpurun_out/gpass_full.ncu-rep gpurun_out/sum_gpass.json "ncu --set full --clock-control none, bench.py --gate 1 (cfg5) --steps 1 --warmup 3: k_psort_scatter, k_gpass 1 and 2" > /dev/null
rm -f gpurun_out/*.ncu-rep
GATE=1 python tools/dbg/n_sweep.py > gpurun_out/n_sweep_gated.json 2> gpurun_out/n_sweep_gated.err; echo nsweep=$?
