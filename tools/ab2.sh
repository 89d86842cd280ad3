#!/bin/bash
# Same-box A/B: main library vs variants over (config, p) cases (development aid).
# Usage: LIBS="a.so b.so" CASES="c3:256 c2c:32768" bash tools/ab2.sh
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for lib in $LIBS; do
  for cp in $CASES; do
    c=${cp%%:*}; p=${cp#*:}
    PFT_LIB=$lib timeout 200 python bench.py --config $c --p $p --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print('$lib'.split('/')[-1], '$c', $p, 'r', d['config']['r'], 'P1', d['config']['P1'], 'P2', d['config']['P2'], 'us', round(d['ms_per_step']*1e3,2), 'GB/s', round(d['input_gbs']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/ab2_${TAG}.log 2>&1
  done
done
done
