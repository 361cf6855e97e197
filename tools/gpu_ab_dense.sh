#!/bin/bash
# A/B of build variants in paper_1503_03769_b200/lib_variants/ on the dense cfg5 bench
mkdir -p gpurun_out
shopt -s nullglob
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  python bench.py --no-gated-leg --no-cpu-baseline --steps 6 > gpurun_out/abd_$n.json 2> gpurun_out/abd_$n.err
  python -c "import json;d=json.load(open('gpurun_out/abd_$n.json'));print('$n',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms'].items() if k in ('pass1','pass2')}, d['clocks']['sm_mhz'])"
done
