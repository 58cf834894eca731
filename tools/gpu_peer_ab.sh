#!/bin/bash
# Interleaved A/B of the cross-process exchange path (PeerStack, world size 1) across builds (args: names).
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default "$@"; do
    if [ $v = default ]; then L=""; else L="RSP_LIB=$PWD/paper_2504_19449_b200/librsparse_b200_$v.so"; fi
    env $L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-dense --check --force-sharded --exchange kernel > gpurun_out/pab_${v}_$rep.json 2>gpurun_out/pab_${v}_$rep.err
    python -c "import json;d=json.loads(open('gpurun_out/pab_${v}_$rep.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), d['check']['ok'])" 2>&1 | tail -1
  done
done
