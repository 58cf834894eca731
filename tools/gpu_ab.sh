#!/bin/bash
# A/B of RSP_KNOBS settings on the default bench line, interleaved (args: knob values; 0 = default).
mkdir -p gpurun_out
for rep in 1 2; do
  for k in "$@"; do
    RSP_KNOBS=$k timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/ab_${k}_$rep.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${k}_$rep.json'));print('knobs=$k', round(d['value'],1), d['config']['step_ms_p10_p50_p90'], d['roofline']['frac'])"
  done
done
