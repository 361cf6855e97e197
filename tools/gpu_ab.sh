#!/bin/bash
# A/B: gated bench for the default build and build variants in paper_1503_03769_b200/lib_variants/
mkdir -p gpurun_out
shopt -s nullglob
[ -n "$SKIP_TESTS" ] || timeout 600 python -m pytest tests/test_gpu_gate.py -x -q > gpurun_out/pytest_gate.log 2>&1; echo gate_tests=$?
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  python bench.py --gate 1 --no-gated-leg --no-cpu-baseline > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$n.json'));print('$n',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms'].items()})"
done
if [ -n "$NCU" ]; then
  unset PHD_LIB
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gate.csv python bench.py --gate 1 --no-gated-leg --no-cpu-baseline --steps 3 > gpurun_out/ncu_gate.log 2>&1; echo ncu=$?
fi
