#!/bin/bash
# One gpurun call: GPU tests, the default bench line, every config, the reference arm, the 2-D
# and anomaly lines, then (each after its plain command exited 0) the ncu launch list and one
# full K1 capture.  Usage on the box: TAG=r02e bash tools/round_run.sh
TAG=${TAG:-rxx}
O=gpurun_out
mkdir -p $O
if [ "${PART:-1}" = 1 ]; then
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_${TAG}.log
timeout 300 python bench.py > $O/bench_default_${TAG}.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_${TAG}.log 2>&1
for c in c1 c2a c2c c3 c4; do
  timeout 600 python bench.py --config $c --no-e2e > $O/bench_${c}_${TAG}.log 2>&1
done
timeout 900 python bench.py --config c5 --no-e2e --steps 30 > $O/bench_c5_${TAG}.log 2>&1
timeout 900 python bench.py --config c5 --force-sharded --steps 20 > $O/bench_c5_sharded_${TAG}.log 2>&1
timeout 600 python tools/bench_2d.py > $O/bench_2d_${TAG}.log 2>&1
timeout 600 python tools/bench_anomaly.py > $O/bench_anomaly_${TAG}.log 2>&1
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-parity --p ${P_C2B:-16384}"
if $CMD > $O/plain_${TAG}.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $O/launches_c2b_${TAG}.csv $CMD > $O/ncu_launch_${TAG}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 6 -c 1 \
    -o $O/prof_k1_c2b_${TAG} $CMD > $O/ncu_k1_${TAG}.log 2>&1
fi
ls -la $O | tail -30
exit 0
fi
C3CMD="python bench.py --config c3 --p 256 --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity"
if $C3CMD > $O/plain_c3_${TAG}.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $O/launches_c3_${TAG}.csv $C3CMD > $O/ncu_launch_c3_${TAG}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 3 -c 1 \
    -o $O/prof_k1_c3_${TAG} $C3CMD > $O/ncu_k1_c3_${TAG}.log 2>&1
fi
C2CCMD="python bench.py --config c2c --p 32768 --steps 20 --warmup 3 --no-e2e --no-cpu --no-parity"
if $C2CCMD > $O/plain_c2c_${TAG}.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $O/launches_c2c_${TAG}.csv $C2CCMD > $O/ncu_launch_c2c_${TAG}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 \
    -o $O/prof_k2_c2c_${TAG} $C2CCMD > $O/ncu_k2_c2c_${TAG}.log 2>&1
fi
ls -la $O | tail -20
