#!/bin/bash
# full GPU suite, then the bench line twice
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/full_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/full_pytest.log
tail -n 2 gpurun_out/full_pytest.log
bash tools/gpu_ab.sh "${@:-0}"
