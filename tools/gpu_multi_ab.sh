#!/bin/bash
# Interleaved bench A/B of the default build against variant builds
# paper_2504_19449_b200/librsparse_b200_<name>.so (args: names).
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default "$@"; do
    if [ $v = default ]; then L=""; else L="RSP_LIB=$PWD/paper_2504_19449_b200/librsparse_b200_$v.so"; fi
    env $L timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense --check > gpurun_out/mab_${v}_$rep.json 2>gpurun_out/mab_${v}_$rep.err
    python -c "import json;d=json.load(open('gpurun_out/mab_${v}_$rep.json'));print('$v', round(d['value'],1), d['config']['step_ms_p10_p50_p90'][1], d['check']['ok'])" 2>&1 | tail -1
  done
done
