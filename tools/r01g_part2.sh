#!/bin/bash
# 2-D bench lines + one ncu capture (C3 K1 or C2c K2), each call under the 64 MiB copy-back limit.
O=gpurun_out; mkdir -p $O; TAG=${TAG:-r01g}
if [ "$WHAT" = c3 ]; then
  timeout 300 python tools/bench_2d.py > $O/bench_2d_${TAG}.log 2>&1
  timeout 300 python tools/bench_2d.py --n1 1024 --n2 16384 --m1 32 --m2 256 --mu1 -77 --mu2 1000 > $O/bench_2d_b_${TAG}.log 2>&1
  C3CMD="python bench.py --config c3 --p 256 --steps 5 --warmup 3 --no-e2e --no-cpu"
  if $C3CMD > $O/plain_c3_${TAG}.log 2>&1; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file $O/launches_c3_${TAG}.csv $C3CMD > $O/ncu_launch_c3_${TAG}.log 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 3 -c 1 \
      -o $O/prof_k1_c3_${TAG} $C3CMD > $O/ncu_k1_c3_${TAG}.log 2>&1
    ncu -i $O/prof_k1_c3_${TAG}.ncu-rep --page raw --csv > $O/prof_k1_c3_${TAG}.raw.csv && rm -f $O/prof_k1_c3_${TAG}.ncu-rep
  fi
else
  C2CCMD="python bench.py --config c2c --p 32768 --steps 20 --warmup 3 --no-e2e --no-cpu"
  if $C2CCMD > $O/plain_c2c_${TAG}.log 2>&1; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file $O/launches_c2c_${TAG}.csv $C2CCMD > $O/ncu_launch_c2c_${TAG}.log 2>&1
    timeout 900 ncu --set full --clock-control none -k regex:k2_ -s 6 -c 1 \
      -o $O/prof_k2_c2c_${TAG} $C2CCMD > $O/ncu_k2_c2c_${TAG}.log 2>&1
    ncu -i $O/prof_k2_c2c_${TAG}.ncu-rep --page raw --csv > $O/prof_k2_c2c_${TAG}.raw.csv && rm -f $O/prof_k2_c2c_${TAG}.ncu-rep
  fi
fi
ls -la $O
