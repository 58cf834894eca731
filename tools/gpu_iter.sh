#!/usr/bin/env bash
# Quick iteration: GPU parity tests (first failure stops), per-linear microbench, phase trace.
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python tools/microbench.py --graph > gpurun_out/microbench_$TAG.txt 2>&1
timeout 300 python tools/trace.py > gpurun_out/trace_$TAG.txt 2>&1
echo done
