#!/bin/bash
# A/B: (build variant x environment) on the dense configs: step, pass1, pass2 ms
#   ENVS="PHD_FORCE_ZL=16;PHD_FORCE_ZL=8" CFGS="cfg5 cfg4" bash tools/gpu_ab_env.sh
mkdir -p gpurun_out
shopt -s nullglob
IFS=';' read -ra EL <<< "${ENVS:-NONE=1}"
for CFG in ${CFGS:-cfg5 cfg4}; do
for v in default paper_1503_03769_b200/lib_variants/*.so; do
for e in "${EL[@]}"; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  tag=${n}_$(echo $e | tr '=' '_')
  env $e python bench.py --config $CFG --no-gated-leg --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/ab_${CFG}_$tag.json 2> gpurun_out/ab_${CFG}_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/ab_${CFG}_$tag.json'));print('$CFG $tag',round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['kernel_ms'].items() if k in ('pass1','pass2','update')}, 'frac',round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_${CFG}_$tag.err
done
done
done
