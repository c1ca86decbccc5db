#!/bin/bash
# one development iteration on the GPU box: GPU tests, a short bench, the
# composition bench, then (only if the plain run passed) ncu of named kernels.
#   bash tools/iter.sh TAG "regex:kernelA|kernelB"
TAG=${1:-it}; KRE=${2:-}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 --no-compose"
$B > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
python bench_compose.py --regime both --instances 2000 --steps 3 --cpu-sample 2 > gpurun_out/${TAG}_compose.log 2>&1; echo "compose rc=$?"
if [ -n "$KRE" ]; then
  ncu --set full --import-source on --clock-control none -k "$KRE" -c 2 -o gpurun_out/${TAG}_ncu \
      python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-config5 --no-compose > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"
fi
