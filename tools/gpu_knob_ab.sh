#!/bin/bash
# Correctness (config-2 stack parity) then interleaved timing of RSP_KNOBS values.
# args: knob values (0 = default)
mkdir -p gpurun_out
for k in "$@"; do
  RSP_KNOBS=$k timeout 600 python -m pytest tests/test_gpu_config2.py -x -q -k stack -p no:cacheprovider > gpurun_out/kab_test_$k.txt 2>&1
  echo "knobs=$k parity: $(tail -1 gpurun_out/kab_test_$k.txt)"
done
for rep in 1 2; do
  for k in "$@"; do
    RSP_KNOBS=$k timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense > gpurun_out/kab_${k}_$rep.json 2>gpurun_out/kab_${k}_$rep.err
    python -c "import json;d=json.load(open('gpurun_out/kab_${k}_$rep.json'));print('knobs=$k', round(d['value'],1), d['config']['step_ms_p10_p50_p90'], round(d['roofline']['frac'],4))"
  done
done
