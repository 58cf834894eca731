#!/bin/bash
# A/B of the default build against librsparse_b200_base.so (the previous kernel, built with
# RSP_NVCC_EXTRA), after the default build's parity tests; then a phase trace of the default build.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab_pytest.txt 2>&1
tail -2 gpurun_out/ab_pytest.txt
for rep in 1 2; do
  for v in new base; do
    if [ $v = new ]; then L=""; else L="RSP_LIB=$PWD/paper_2504_19449_b200/librsparse_b200_base.so"; fi
    env $L timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense --check > gpurun_out/ab_${v}_$rep.json 2>gpurun_out/ab_${v}_$rep.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$rep.json'));print('$v', round(d['value'],1), d['config']['step_ms_p10_p50_p90'], d['check']['ok'])" 2>&1 | tail -1
  done
done
timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/ab_trace.txt 2>&1
head -12 gpurun_out/ab_trace.txt
