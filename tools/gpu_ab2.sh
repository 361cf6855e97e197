#!/bin/bash
# A/B of build variants (lib_variants/*.so vs default) on cfg5 and cfg4 dense: step, pass1, pass2 ms
mkdir -p gpurun_out
shopt -s nullglob
for CFG in ${CFGS:-cfg5 cfg4}; do
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  python bench.py --config $CFG --no-gated-leg --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/ab_${CFG}_$n.json 2> gpurun_out/ab_${CFG}_$n.err
  python -c "import json;d=json.load(open('gpurun_out/ab_${CFG}_$n.json'));print('$CFG $n',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms'].items() if k in ('pass1','pass2','predict','resample')}, 'frac',round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/ab_${CFG}_$n.err
done
done
