#!/bin/bash
# Per-linear microbench (config 0 fp32, config 1 bf16 shapes, config-2 rho 0.5 plans) and a one-layer stack trace.
mkdir -p gpurun_out
timeout 600 python tools/microbench.py --shapes q --rho 0 --s 0.5 --wdt f32 --xdt f32 --graph > gpurun_out/ev_config0.jsonl 2>&1
timeout 900 python tools/microbench.py --shapes q,gate,down --rho 0 --s 0.5 --graph > gpurun_out/ev_config1.jsonl 2>&1
timeout 900 python tools/microbench.py --shapes q,gate,down --graph > gpurun_out/ev_config2rho05.jsonl 2>&1
timeout 300 python tools/stack_trace.py --layers 1 > gpurun_out/ev_trace.txt 2>&1
cat gpurun_out/ev_config0.jsonl gpurun_out/ev_config1.jsonl gpurun_out/ev_config2rho05.jsonl | cut -c1-250; head -3 gpurun_out/ev_trace.txt
