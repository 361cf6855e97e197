#!/bin/bash
# One gpurun call worth of evidence: smoke, GPU tests, bench (cfg5 + cfg3/cfg4), ncu launch list, ncu --set full of the update passes.
mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench=$?
for c in cfg3 cfg4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass --launch-skip 6 -c 2 -o gpurun_out/pass_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
