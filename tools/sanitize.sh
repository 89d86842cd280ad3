#!/bin/bash
# compute-sanitizer over every device form (tools/sanitize.py); logs under gpurun_out/.
O=gpurun_out; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize.py > $O/sanitize_plain.log 2>&1; echo "plain exit $?" >> $O/sanitize_plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $t --print-limit 20 python tools/sanitize.py > $O/sanitize_$t.log 2>&1
  echo "$t exit $?" >> $O/sanitize_$t.log
done
tail -n 4 $O/sanitize_*.log
