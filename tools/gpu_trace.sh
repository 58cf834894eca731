#!/usr/bin/env bash
TAG=${1:-tr}
mkdir -p gpurun_out
timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/stack_trace_${TAG}.txt 2>&1
echo done
