#!/usr/bin/env bash
TAG=${1:-p2}
mkdir -p gpurun_out
timeout 300 ./tools/overhead_probe > gpurun_out/overhead_probe_$TAG.txt 2>&1
timeout 300 ./tools/gather_probe > gpurun_out/gather_probe_$TAG.txt 2>&1
echo done
