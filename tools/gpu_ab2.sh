#!/bin/bash
# stack parity subset, then an A/B of knob settings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stack or bench or forward" > gpurun_out/ab2_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/ab2_pytest.log
tail -n 2 gpurun_out/ab2_pytest.log
bash tools/gpu_ab.sh "$@"
