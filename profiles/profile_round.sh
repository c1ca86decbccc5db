#!/bin/bash
# Round profile capture: bench line, launch list, DRAM traffic and ncu full of the top kernels.
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prof_launch.log 2>&1
rm -f gpurun_out/prof_dram.csv
for k in jffc_sim exp_streams row_stats; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      -k regex:$k -c 1 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline 2>/dev/null \
      | grep -v "^==" | (if [ -f gpurun_out/prof_dram.csv ]; then tail -n +2; else cat; fi) >> gpurun_out/prof_dram.csv
done
ncu --set full --import-source on --clock-control none -k regex:"jffc_sim|row_stats" -c 1 \
    -o gpurun_out/prof_full python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prof_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:row_stats -c 1 \
    -o gpurun_out/prof_full_stats python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prof_full2.log 2>&1
echo done
