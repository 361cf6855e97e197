#!/bin/bash
# per-kernel mean durations (ncu launch list) for each build variant: CFG, ARGS, KREGEX
mkdir -p gpurun_out
shopt -s nullglob
CFG=${CFG:-cfg5}; KREGEX=${KREGEX:-.}
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$KREGEX" --csv --log-file gpurun_out/kl_${CFG}_$n.csv \
    python bench.py --config $CFG --no-gated-leg --no-cpu-baseline --steps 3 $ARGS > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/kl_${CFG}_$n.csv gpurun_out/kl_${CFG}_$n.txt > /dev/null 2>&1
  echo "== $CFG $n"; sed -n '4,12p' gpurun_out/kl_${CFG}_$n.txt
done
