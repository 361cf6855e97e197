#!/bin/bash
# gated-update bring-up: build, gated GPU tests, dense parity subset, bench with the gated leg
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_gate.py -x -q > gpurun_out/pytest_gate.log 2>&1; echo gate_tests=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "update_parity or stagewise" > gpurun_out/pytest_dense.log 2>&1; echo dense_tests=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_gate.json 2> gpurun_out/bench_gate.err; echo bench=$?
timeout 300 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_gate_cfg4.json 2> gpurun_out/bench_gate_cfg4.err; echo bench4=$?
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/bench_gate_cfg3.json 2> gpurun_out/bench_gate_cfg3.err; echo bench3=$?
