#!/usr/bin/env bash
# One full ncu capture (high-rate stall sampling) of the 1-layer stack launch
# from tools/stack_trace.py (after warm-up launches).
TAG=${1:-n1}
mkdir -p gpurun_out
timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/ncu_plain_$TAG.log 2>&1 &&
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
    -k regex:stack_kernel -s 10 -c 1 -o gpurun_out/one_$TAG python tools/stack_trace.py --layers 1 \
    > gpurun_out/ncu_one_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/ncu_one_$TAG.log
