#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pf_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pf_pytest.log
tail -n 2 gpurun_out/pf_pytest.log
bash tools/gpu_ab.sh 0 4096
timeout 300 python tools/batch_bench.py --batches 2,4,8,16 > gpurun_out/pf_batch.log 2>&1; cat gpurun_out/pf_batch.log
