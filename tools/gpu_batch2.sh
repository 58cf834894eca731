#!/bin/bash
# batched path: parity (default and tcgen05), config-3 timing, phase trace.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch or bench" > gpurun_out/b2_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/b2_pytest.log
RSP_BATCH_TC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k batch > gpurun_out/b2_pytest_tc.log 2>&1
echo "pytest-tc exit $?" >> gpurun_out/b2_pytest_tc.log
timeout 300 python tools/batch_bench.py --batches 2,4,8,16 > gpurun_out/b2_bench.log 2>&1
RSP_BATCH_PDL=0 timeout 300 python tools/batch_bench.py --batches 2,16 > gpurun_out/b2_bench_nopdl.log 2>&1
#timeout 300 python tools/batch_trace.py > gpurun_out/b2_trace.log 2>&1
tail -n 2 gpurun_out/b2_pytest.log gpurun_out/b2_pytest_tc.log; cat gpurun_out/b2_bench.log gpurun_out/b2_bench_nopdl.log gpurun_out/b2_trace.log
