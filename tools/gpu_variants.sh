#!/usr/bin/env bash
TAG=${1:-var}
mkdir -p gpurun_out
out=gpurun_out/variants_$TAG.txt
: > $out
for v in "" "RSP_SMEM_OPS=1 RSP_KNOBS=12" "RSP_SMEM_OPS=1 RSP_KNOBS=8" ""; do
  echo "== $v" >> $out
  env $v timeout 300 python bench.py --no-cpu --no-dense --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'us/token', round(d['roofline']['frac'],3))" >> $out 2>&1
done
RSP_SMEM_OPS=1 RSP_KNOBS=12 timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/stack_trace_$TAG.txt 2>&1
echo done
