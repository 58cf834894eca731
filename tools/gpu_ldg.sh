#!/usr/bin/env bash
# Rebuild with each streaming-load variant and bench it (experiment).
out=gpurun_out/ldg_variants.txt
: > $out
for v in 0 1 2 0; do
  RSP_NVCC_EXTRA="-DRSP_LDG=$v" python -m paper_2504_19449_b200.build --force > /dev/null 2>&1
  echo "== RSP_LDG=$v" >> $out
  timeout 300 python bench.py --no-cpu --no-dense --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'us/token', round(d['roofline']['frac'],3))" >> $out 2>&1
done
