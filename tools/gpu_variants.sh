#!/usr/bin/env bash
# Short bench of the stack under environment variants (first line: default).
TAG=${1:-var}
mkdir -p gpurun_out
out=gpurun_out/variants_$TAG.txt
: > $out
for v in "" "RSP_NO_SMEM_OPS=1" "RSP_KNOBS=2" "RSP_MAX_KSPLITS=12" "RSP_MAX_KSPLITS=48"; do
  echo "== $v" >> $out
  env $v timeout 300 python bench.py --no-cpu --no-dense --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'us/token', round(d['roofline']['frac'],3))" >> $out 2>&1
done
echo done
