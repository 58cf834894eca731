#!/bin/bash
# Selected GPU tests: bash tools/gpu_some.sh <pytest args...>
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -p no:cacheprovider "$@" > gpurun_out/s_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/s_pytest.txt
tail -3 gpurun_out/s_pytest.txt
