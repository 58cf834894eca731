#!/usr/bin/env bash
# GPU parity tests, then bench + stack-trace variants (env settings as args).
TAG=${1:-it}
shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
bash tools/gpu_var2.sh $TAG "$@"
