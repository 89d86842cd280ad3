#!/bin/bash
# GPU tests + quick bench lines for a list of configs (+ optional ncu of one config's K1).
# Usage: TAG=x CFGS="c3 c2c" NCU_CFG="c3 --p 256" bash tools/check_run.sh
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_${TAG}.log 2>&1; echo "exit $?" >> $O/pytest_gpu_${TAG}.log
for c in ${CFGS:-c2b}; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 > $O/bench_${c}_${TAG}.json
done
if [ -n "$NCU_CFG" ]; then
  CMD="python bench.py --config $NCU_CFG --steps 5 --warmup 3 --no-e2e --no-cpu"
  $CMD > $O/plain_ncu_${TAG}.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 3 -c 1 -o $O/prof_k1_${TAG} $CMD > $O/ncu_${TAG}.log 2>&1
fi
ls $O | tail -3
