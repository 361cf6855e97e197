#!/bin/bash
# round-2 check: all GPU tests (near-tie log) + default bench cfg5 + cfg4
mkdir -p gpurun_out
export PHD_NEAR_TIE_LOG=gpurun_out/near_ties.json
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo gpu_tests=$?
tail -30 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
python bench.py --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench=$?
python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4=$?
fi
