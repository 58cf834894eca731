#!/bin/bash
# The GPU parity suite on the bounds-checked build (librsparse_b200_debug.so, built with
# RSP_NVCC_EXTRA=-DRSP_DEBUG_CHECKS=1): compute-sanitizer is closed on the GPU pool, so the
# stack kernel checks its own shared-memory carve-up, plan and workspace indices and traps.
mkdir -p gpurun_out
RSP_LIB=$PWD/paper_2504_19449_b200/librsparse_b200_debug.so timeout 1500 python -m pytest tests -m gpu -x -q \
   -p no:cacheprovider -k "not sharded_bench_path and not integration" > gpurun_out/dbg_pytest.txt 2>&1
echo "debug-checks pytest rc=$?" >> gpurun_out/dbg_pytest.txt
RSP_LIB=$PWD/paper_2504_19449_b200/librsparse_b200_debug.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-dense --check > gpurun_out/dbg_bench.json 2>&1
echo "debug-checks bench rc=$?" >> gpurun_out/dbg_pytest.txt
tail -3 gpurun_out/dbg_pytest.txt; head -c 300 gpurun_out/dbg_bench.json
