#!/bin/bash
# K2 tail (K2's work by K1's last arrivals) vs the separate K2 grid, within one box.
# Usage on the box: TAG=x bash tools/k2tail_ab.sh
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k2_tail or tail_forms or second_pass or forms_agree" \
  > $O/pytest_k2tail_${TAG}.log 2>&1; echo "exit $?" >> $O/pytest_k2tail_${TAG}.log
for cfg in "c2c --p 32768" "c5 --steps 60"; do
  for t in off on; do
    timeout 300 python bench.py --config $cfg --k2-tail $t --no-e2e --no-cpu 2>/dev/null | tail -1 \
      > $O/ab_${cfg%% *}_${t}_${TAG}.json
  done
done
for L in 16 32 128; do
  timeout 300 python bench.py --config c2c --p 32768 --k2-tail on --reducers $L --no-e2e --no-cpu 2>/dev/null | tail -1 \
    > $O/ab_c2c_L${L}_${TAG}.json
done
timeout 300 python bench.py --config c2c --k2-tail on --no-e2e --no-cpu 2>/dev/null | tail -1 > $O/ab_c2c_auto_${TAG}.json
for f in $O/ab_*_${TAG}.json; do echo "$f $(python -c "import json,sys; d=json.load(open('$f')); print(round(d['ms_per_step']*1e3,2), 'us', d['config']['p'], d['config']['tail'])" 2>&1 | tail -1)"; done
