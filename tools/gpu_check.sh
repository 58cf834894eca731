#!/usr/bin/env bash
# One gpurun call: smoke, GPU parity tests, the default bench line, then (only
# after the bench exited 0 without a profiler) the ncu launch list of the
# timed steps and a full capture of one stack-kernel launch.
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag]'
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --check > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench exit $?" >> $OUT/bench_$TAG.err
timeout 1200 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
PROF="python bench.py --steps 3 --warmup 3 --profile"
timeout 600 $PROF > $OUT/prof_plain_$TAG.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/launches_$TAG.csv $PROF > $OUT/ncu_launches_$TAG.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:stack_kernel -s 3 -c 1 \
      -o $OUT/prof_$TAG $PROF > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu exit $?" >> $OUT/prof_plain_$TAG.log
