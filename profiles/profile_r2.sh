#!/bin/bash
# Round-2 profile capture (one gpurun call, 1 GPU, config 2 + config 4):
#   prof_launches.csv   every launch of one short bench run with its device time,
#                       executed instructions, DRAM bytes and SM cycles
#   prof_seg.ncu-rep    ncu --set full of the segmented simulator
#   prof_stats.ncu-rep  ncu --set full of the row-statistics pass
#   prof_streams.ncu-rep ncu --set full of the stream (+ prefix) kernel
#   prof_compose_{moderate,full}.ncu-rep ncu --set full of gbp_kernel and gca_kernel (config 4, 2000 instances)
# Each ncu command follows the same command line run plain (exit 0) first.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-config5 --no-compose"
$B > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/prof_launches.csv $B > gpurun_out/prof_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:jffc_seg_kernel -c 1 \
    -o gpurun_out/prof_seg $B > gpurun_out/prof_seg.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:row_stats -c 1 \
    -o gpurun_out/prof_stats $B > gpurun_out/prof_stats.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:exp_streams -c 1 \
    -o gpurun_out/prof_streams $B > gpurun_out/prof_streams.log 2>&1
for R in moderate full; do
  C="python bench_compose.py --regime $R --instances 2000 --steps 1 --cpu-sample 1"
  $C > gpurun_out/prof_compose_${R}_plain.log 2>&1 || exit 1
  ncu --set full --import-source on --clock-control none -k regex:"gbp_kernel|gca_kernel|gca_warp_kernel" -c 2 \
      -o gpurun_out/prof_compose_$R $C > gpurun_out/prof_compose_$R.log 2>&1
done
echo done
