#!/usr/bin/env bash
# Quick iteration: GPU parity tests (default + shared-memory operands), stack trace, bench variants.
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
RSP_SMEM_OPS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stack or config1 or ragged" > gpurun_out/pytest_gpu_smem_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_smem_$TAG.log
timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/stack_trace_$TAG.txt 2>&1
out=gpurun_out/variants_$TAG.txt
: > $out
for v in ""; do
  echo "== $v" >> $out
  env $v timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'us/token', round(d['roofline']['frac'],3), 'cublas', round(d.get('dense_cublas_us_per_token',0),1), 'inhouse-dense', round(d.get('dense_inhouse_us_per_token',0),1))" >> $out 2>&1
done
echo done
