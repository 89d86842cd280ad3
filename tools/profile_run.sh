#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): plain run first, then ncu on the same command.
set -x
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches${TAG}.csv $CMD > gpurun_out/ncu_launch${TAG}.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 4 -c 1 -o gpurun_out/prof_k1${TAG} $CMD > gpurun_out/ncu_k1${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_ -s 4 -c 1 -o gpurun_out/prof_k2${TAG} $CMD > gpurun_out/ncu_k2${TAG}.log 2>&1
ls -la gpurun_out
