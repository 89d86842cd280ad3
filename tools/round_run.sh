#!/bin/bash
# One gpurun call: GPU tests, the default bench line, every config, the reference arm,
# then (each after its plain command exited 0) the ncu launch list and one full K1 capture.
# Usage on the box: TAG=r01d bash tools/round_run.sh
TAG=${TAG:-rxx}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_${TAG}.log
timeout 300 python bench.py > $O/bench_default_${TAG}.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_${TAG}.log 2>&1
for c in c1 c2a c2c c3 c4 c5; do
  timeout 300 python bench.py --config $c --no-e2e > $O/bench_${c}_${TAG}.log 2>&1
done
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu"
if $CMD > $O/plain_${TAG}.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $O/launches_c2b_${TAG}.csv $CMD > $O/ncu_launch_${TAG}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 6 -c 1 \
    -o $O/prof_k1_c2b_${TAG} $CMD > $O/ncu_k1_${TAG}.log 2>&1
fi
ls -la $O
