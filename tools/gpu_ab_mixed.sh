#!/bin/bash
# A/B of build variants on the gated cfg-5 step: step, gated pass 1/2, resampling leg (ms),
# each variant run REPS times in alternation (box-to-box noise stays out of the comparison)
mkdir -p gpurun_out
shopt -s nullglob
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ab_tests.log; fi
for r in $(seq ${REPS:-2}); do
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  python bench.py --config ${CFG:-cfg5} --gate ${GATE:-1} --no-gated-leg --no-cpu-baseline --steps ${STEPS:-10} > gpurun_out/abm_$n.json 2> gpurun_out/abm_$n.err
  python -c "import json;d=json.load(open('gpurun_out/abm_$n.json'));k=d['kernel_ms'];print('rep $r $n step',round(d['ms_per_step'],4),'p1',round(k['pass1'],4),'p2',round(k['pass2'],4),'res',round(d['hbm_kernels']['resample']['ms'],4),round(d['hbm_kernels']['resample']['frac'],3),d['clocks']['sm_mhz'])" || tail -5 gpurun_out/abm_$n.err
done
done
