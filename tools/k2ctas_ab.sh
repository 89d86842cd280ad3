#!/bin/bash
# C2c: K2 grid width sweep (narrow looping K2 FFT grid) and K2 tail; C5 tail on/off.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k2_tail or tail_forms or second_pass or forms_agree" \
  > $O/pytest_k2_${TAG}.log 2>&1; echo "exit $?" >> $O/pytest_k2_${TAG}.log
for kc in 0 24 40 48 64; do
  timeout 300 python bench.py --config c2c --p 32768 --k2-tail off --k2-ctas $kc --no-e2e --no-cpu 2>/dev/null | tail -1 \
    > $O/ab_c2c_kc${kc}_${TAG}.json
done
timeout 300 python bench.py --config c2c --no-e2e --no-cpu 2>/dev/null | tail -1 > $O/ab_c2c_auto_${TAG}.json
for t in off on auto; do
  timeout 300 python bench.py --config c5 --steps 60 --k2-tail $t --no-e2e --no-cpu 2>/dev/null | tail -1 > $O/ab_c5_${t}_${TAG}.json
done
for f in $O/ab_*_${TAG}.json; do echo "$f $(python -c "import json,sys; d=json.load(open('$f')); print(round(d['ms_per_step']*1e3,2), 'us', d['config']['p'], d['config']['tail'])" 2>&1 | tail -1)"; done
