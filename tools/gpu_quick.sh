#!/bin/bash
# quick A/B: stack parity subset, then the default bench line twice.
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stack or bench or smoke or forward" > gpurun_out/q_pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/q_pytest_$TAG.log
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/q_bench_${TAG}_$i.json 2>/dev/null; done
tail -n 2 gpurun_out/q_pytest_$TAG.log
for i in 1 2; do python -c "import json;d=json.load(open('gpurun_out/q_bench_${TAG}_$i.json'));print(d['value'],d['config']['step_ms_p10_p50_p90'],d['clocks']['sm_mhz'])"; done
