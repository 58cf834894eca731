#!/usr/bin/env bash
# Bench variants (env knobs) + a stack trace per variant.
TAG=${1:-var}
shift
mkdir -p gpurun_out
out=gpurun_out/variants_$TAG.txt
: > $out
i=0
for v in "$@"; do
  echo "== $v" >> $out
  env $v timeout 300 python bench.py --no-cpu --no-dense --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'us/token', round(d['roofline']['frac'],3))" >> $out 2>&1
  env $v timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/stack_trace_${TAG}_$i.txt 2>&1
  i=$((i+1))
done
echo done
