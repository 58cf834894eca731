#!/bin/bash
# Full GPU test suite + host facts of the box.
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20) > gpurun_out/t_host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/t_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/t_pytest.txt
tail -3 gpurun_out/t_pytest.txt
