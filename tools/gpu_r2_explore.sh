#!/bin/bash
# Round-2 exploration: baseline bench, operand-preload variants, phase traces.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/x_smi.txt 2>&1
python -c "import paper_2504_19449_b200 as r; r.lib()" > gpurun_out/x_import.txt 2>&1
for rep in 1 2; do
for e in "-" "RSP_SMEM_OPS=1" "RSP_SMEM_OPS=1 RSP_OBUF_KB=48" "RSP_SMEM_OPS=1 RSP_KNOBS=4"; do
  if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
  tag=$(echo "$e" | tr ' =' '__')
  env $envs timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense > gpurun_out/x_$tag.$rep.json 2>gpurun_out/x_$tag.$rep.err
  python -c "import json;d=json.load(open('gpurun_out/x_$tag.$rep.json'));print('[$e]', round(d['value'],1), d['config']['step_ms_p10_p50_p90'])" 2>&1 | tail -1
done
done
timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/x_trace_default.txt 2>&1
RSP_SMEM_OPS=1 timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/x_trace_smemops.txt 2>&1
echo done
