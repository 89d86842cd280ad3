#!/bin/bash
# Quick GPU-box pass: GPU tests, then the default bench line and a few configs (no ncu).
# Usage on the box: TAG=r02b CONFIGS="c2c c5" bash tools/gpu_check.sh
TAG=${TAG:-rxx}
O=gpurun_out
mkdir -p $O
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $O/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu_${TAG}.log
timeout 300 python bench.py > $O/bench_default_${TAG}.log 2>&1
for c in ${CONFIGS}; do
  timeout 600 python bench.py --config $c --no-e2e ${BENCH_ARGS} > $O/bench_${c}_${TAG}.log 2>&1
done
for c in ${SHARDED}; do
  timeout 600 python bench.py --config $c --force-sharded --steps 20 > $O/bench_${c}_sharded_${TAG}.log 2>&1
done
ls -la $O | tail -20
