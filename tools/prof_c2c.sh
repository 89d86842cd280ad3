#!/bin/bash
# C2c (chained, K2 workers inside K1's grid): plain run, ncu launch list, one full capture of K1.
TAG=${TAG:-rxx}
O=gpurun_out
mkdir -p $O
CMD="python bench.py --config c2c --p 32768 --steps 20 --warmup 3 --no-e2e --no-cpu --no-parity"
if $CMD > $O/plain_c2c_${TAG}.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $O/launches_c2c_${TAG}.csv $CMD > $O/ncu_launch_c2c_${TAG}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 30 -c 1 \
    -o $O/prof_k1_c2c_${TAG} $CMD > $O/ncu_k1_c2c_${TAG}.log 2>&1
fi
ls -la $O | tail -8
