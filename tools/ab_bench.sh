#!/bin/bash
# Same-box A/B of bench modes, interleaved (development aid).
for rep in 1 2; do
  for mode in "--streams 1" "--streams 1 --no-pdl" "--streams 2" "--streams 2 --no-pdl"; do
    python bench.py --no-cpu --no-e2e $mode 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$mode', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,2), 'lat', round(d['latency_us_single_stream'],2), 'k1_us', round(d['roofline']['k1_ms']*1e3,2), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
