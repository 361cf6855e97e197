#!/bin/bash
# psort_scatter timing per build variant under ncu (kernel duration + memory metrics)
mkdir -p gpurun_out
shopt -s nullglob
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_drain_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
for v in default paper_1503_03769_b200/lib_variants/*.so; do
  if [ $v = default ]; then unset PHD_LIB; n=default; else export PHD_LIB=$PWD/$v; n=$(basename $v .so); fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"k_psort_scatter|k_ms_hist" --launch-skip 8 -c 4 --csv \
    python bench.py --gate 1 --steps 2 --warmup 3 --no-gated-leg --no-cpu-baseline > gpurun_out/psort_$n.csv 2> gpurun_out/psort_$n.err
  echo $n=$?
done
