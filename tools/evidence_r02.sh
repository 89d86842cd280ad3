#!/bin/bash
# Round-2 evidence: C2b bench with >= 8x L2 input rotation; the 20-step graph profiled as one unit
# (ncu --graph-profiling graph: DRAM bytes of the whole chain); an isolated C2b execute (cluster
# split K1) under --set full.
O=gpurun_out; mkdir -p $O
timeout 300 python bench.py --no-e2e > $O/ev_bench_c2b.log 2>&1
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-parity --p 16384"
if $CMD > $O/ev_plain.log 2>&1; then
  timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/ev_graph.csv $CMD > $O/ev_graph.log 2>&1
fi
if python tools/prof_one.py c2b "" 3 > $O/ev_iso_plain.log 2>&1; then
  timeout 900 ncu --set full --clock-control none -k regex:k1_contract -s 2 -c 1 -o $O/prof_k1_iso_c2b \
    python tools/prof_one.py c2b "" 3 > $O/ev_iso_ncu.log 2>&1
fi
ls -la $O | tail -8
