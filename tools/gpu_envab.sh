#!/bin/bash
# A/B of environment settings on the default bench line (args: "VAR=v VAR2=w" strings; "-" = none)
mkdir -p gpurun_out
i=0
for rep in 1 2; do
  for e in "$@"; do
    i=$((i+1))
    if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
    env $envs timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/envab_$i.json 2>gpurun_out/envab_$i.err
    python -c "import json;d=json.load(open('gpurun_out/envab_$i.json'));print('[$e]', round(d['value'],1), d['config']['step_ms_p10_p50_p90'])" 2>&1 | tail -1
  done
done
