#!/bin/bash
# Multi-GPU evidence on an N-GPU box: the NCCL tests, then the bench at N
# (torchrun, one rank per GPU), as the driver launches it.
#   bash tools/mgpu.sh N
N=${1:-2}
mkdir -p gpurun_out
python -m pytest tests/test_multigpu.py -q > gpurun_out/mgpu_tests_n$N.log 2>&1; echo "tests rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/mgpu_bench_n$N.log 2>&1; echo "bench rc=$?"
