#!/bin/bash
# tcgen05 batched ring path: parity with RSP_BATCH_TC=1, then config-3 timing with and without.
mkdir -p gpurun_out
export RSP_BATCH_TC=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k batch > gpurun_out/tc_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/tc_pytest.log
timeout 300 python tools/batch_bench.py --batches 2,4,8,16 > gpurun_out/tc_bench_on.log 2>&1
RSP_BATCH_TC=0 timeout 300 python tools/batch_bench.py --batches 2,4,8,16 > gpurun_out/tc_bench_off.log 2>&1
tail -3 gpurun_out/tc_pytest.log; cat gpurun_out/tc_bench_on.log gpurun_out/tc_bench_off.log
