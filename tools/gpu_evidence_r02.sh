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
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate_floor.csv python bench.py --gate 1 --gate-floor -71 --no-gated-leg --no-cpu-baseline > gpurun_out/ncu_gate_floor.log 2>&1; echo ncu3=$?
CFGS="cfg5 cfg4" bash tools/gpu_ncu_passes.sh
bash tools/gpu_ncu_hbm.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gpass --launch-skip 4 -c 2 -f -o gpurun_out/gpass_full python bench.py --gate 1 --no-gated-leg --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_gpass.log 2>&1; echo ncu_gpass=$?
# summarise the ncu reports on the box (the .ncu-rep files exceed gpurun's 64 MiB pull limit)
python tools/ncu_summary.py full gpurun_out/pass_full_cfg5.ncu-rep gpurun_out/sum_passes_cfg5.json "ncu --set full --clock-control none, bench.py --config cfg5 --steps 1 --warmup 3: k_pass 1 and 2 of the 4th step" > /dev/null
python tools/ncu_summary.py full gpurun_out/pass_full_cfg4.ncu-rep gpurun_out/sum_passes_cfg4.json "ncu --set full --clock-control none, bench.py --config cfg4 --steps 1 --warmup 3: k_pass 1 and 2 of the 4th step" > /dev/null
python tools/ncu_summary.py full gpurun_out/hbm_full.ncu-rep gpurun_out/sum_hbm.json "ncu --set full --clock-control none, bench.py (cfg5) --steps 1 --warmup 3: k_predict, k_records, k_scan_chunks, k_resample_gather" > /dev/null
python tools/ncu_summary.py full gpurun_out/gpass_full.ncu-rep gpurun_out/sum_gpass.json "ncu --set full --clock-control none, bench.py --gate 1 (cfg5) --steps 1 --warmup 3: k_gpass 1 and 2" > /dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
