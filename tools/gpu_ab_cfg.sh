#!/bin/bash
# A/B of build variants in paper_1503_03769_b200/lib_variants/ on one config:
#   CFG=cfg3 ARGS="--gate 0" REPS=3 bash tools/gpu_ab_cfg.sh
mkdir -p gpurun_out
shopt -s nullglob
CFG=${CFG:-cfg5}; REPS=${REPS:-1}
for rep in $(seq 1 $REPS); do
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  python bench.py --config $CFG --no-gated-leg --no-cpu-baseline $ARGS > gpurun_out/abc_${CFG}_$n.json 2> gpurun_out/abc_${CFG}_$n.err
  python -c "import json;d=json.load(open('gpurun_out/abc_${CFG}_$n.json'));print('$CFG $n',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['kernel_ms'].items()})"
done
done
