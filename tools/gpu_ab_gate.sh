#!/bin/bash
# A/B of build variants on the gated cfg-5 step (bench.py --gate 1): step, gated pass 1/2 ms
mkdir -p gpurun_out
shopt -s nullglob
for CFG in ${CFGS:-cfg5}; do
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  python bench.py --config $CFG --gate 1 --no-gated-leg --no-cpu-baseline --steps ${STEPS:-10} > gpurun_out/abg_${CFG}_$n.json 2> gpurun_out/abg_${CFG}_$n.err
  python -c "import json;d=json.load(open('gpurun_out/abg_${CFG}_$n.json'));print('$CFG gated $n',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms'].items()})" || tail -5 gpurun_out/abg_${CFG}_$n.err
done
done
