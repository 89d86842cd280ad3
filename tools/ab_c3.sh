#!/bin/bash
# C3 A/B: the current library vs variants/lib_nosplit.so (before the small-P2 last-arrival
# reduction), interleaved on one box; then the PFT_TIMELINE per-CTA phases.
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_${TAG:-x}.log 2>&1; echo "exit $?" >> $O/pytest_${TAG:-x}.log
for rep in 1 2; do
  for lib in main nosplit; do
    if [ $lib = main ]; then unset PFT_LIB; else export PFT_LIB=variants/lib_$lib.so; fi
    for c in "c3 --p 256" "c1 --p 2048" "c4 --p 11520" "c2b --p 16384"; do
      v=$(timeout 200 python bench.py --config $c --steps 300 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])")
      echo "$rep $lib ${c%% *} $v" >> $O/ab_c3_${TAG:-x}.txt
    done
  done
done
unset PFT_LIB
PFT_LIB=variants/lib_tl.so timeout 200 python tools/timeline_c3b.py > $O/tl_c3b_fast.txt 2>&1
