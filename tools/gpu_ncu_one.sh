#!/usr/bin/env bash
# Parity tests, then one full ncu capture (high-rate stall sampling) of the 1-layer stack launch.
TAG=${1:-n1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2>/dev/null
timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/ncu_plain_$TAG.log 2>&1 &&
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
    -k regex:stack_kernel -s 10 -c 1 -o gpurun_out/one_$TAG python tools/stack_trace.py --layers 1 \
    > gpurun_out/ncu_one_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/ncu_one_$TAG.log
