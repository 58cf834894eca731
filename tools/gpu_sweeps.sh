#!/bin/bash
# Config 3 (batch 1..16) and config 4 (Llama-3-8B sparsity x rank) sweeps with the current build.
mkdir -p gpurun_out
timeout 1500 python tools/batch_bench.py --batches 1,2,3,4,5,6,8,16 > gpurun_out/sw_config3.jsonl 2> gpurun_out/sw_config3.err
echo "config3 rc=$?"; tail -6 gpurun_out/sw_config3.jsonl | cut -c1-300
timeout 2400 python tools/config4_sweep.py > gpurun_out/sw_config4.jsonl 2> gpurun_out/sw_config4.err
echo "config4 rc=$?"; tail -3 gpurun_out/sw_config4.jsonl | cut -c1-300
