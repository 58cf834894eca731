#!/usr/bin/env bash
TAG=${1:-tr}
mkdir -p gpurun_out
timeout 300 python tools/stack_trace.py --layers 2 > gpurun_out/stack_trace_$TAG.txt 2>&1
RSP_NO_SMEM_OPS=1 timeout 300 python tools/stack_trace.py --layers 2 > gpurun_out/stack_trace_${TAG}_nosmem.txt 2>&1
echo done
