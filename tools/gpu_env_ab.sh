#!/bin/bash
# Parity of selected env settings (PARITY="envA;envB"), then interleaved
# timing of every env setting given as an argument ("-" = none).
mkdir -p gpurun_out
IFS=';' read -ra PAR <<< "${PARITY:-}"
for e in "${PAR[@]}"; do
  [ -z "$e" ] && continue
  env $e timeout 900 python -m pytest tests/test_gpu_config2.py tests/test_gpu_parity.py -x -q -k "stack or config2" -p no:cacheprovider > "gpurun_out/eab_par_$(echo $e | tr ' =' '__').txt" 2>&1
  echo "[$e] parity: $(tail -1 "gpurun_out/eab_par_$(echo $e | tr ' =' '__').txt")"
done
i=0
for rep in 1 2; do
  for e in "$@"; do
    i=$((i+1))
    if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
    env $envs timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense > gpurun_out/eab_$i.json 2>gpurun_out/eab_$i.err
    python -c "import json;d=json.load(open('gpurun_out/eab_$i.json'));print('[$e]', round(d['value'],1), d['config']['step_ms_p10_p50_p90'])" 2>&1 | tail -1
  done
done
