#!/bin/bash
# ncu --set full of the dense passes (k_pass 1 and 2) of cfg 4 and cfg 5 (one step after warm-up)
mkdir -p gpurun_out
for c in ${CFGS:-cfg4 cfg5}; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass --launch-skip 6 -c 2 -f -o gpurun_out/pass_full_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-gated-leg > gpurun_out/ncu_full_$c.log 2>&1; echo ncu_$c=$?
done
