#!/bin/bash
# PDL on/off A/B on step time (cfg5/cfg4 gated, cfg3/cfg2 dense) + the GPU tests with PDL on
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo tests=$?; tail -1 gpurun_out/pytest_gpu.log
for pdl in 1 0; do
  export PHD_PDL=$pdl
  for c in cfg5:1 cfg4:1 cfg3:0 cfg2:0; do
    cfg=${c%:*}; g=${c#*:}
    python bench.py --config $cfg --gate $g --no-gated-leg --no-cpu-baseline > gpurun_out/pdl_${pdl}_$cfg.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/pdl_${pdl}_$cfg.json'));print('pdl=$pdl $cfg gate=$g',round(d['ms_per_step'],4))"
  done
done
