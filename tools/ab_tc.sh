#!/bin/bash
# Same-box A/B of K1 tensor-core variants over the configs (development aid).
O=gpurun_out; mkdir -p $O
./tools/ubench/dmma > $O/dmma2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_tc.log 2>&1; echo "exit $?" >> $O/pytest_gpu_tc.log
for rep in 1 2; do
for lib in paper_2008_12559_b200/libpft_b200.so tools/_variants/lib_tcoff.so tools/_variants/lib_tc8.so; do
  for cp in ${AB_CASES:-"c3 256" "c3 512" "c3 1024" "c2c 32768" "c4 11520" "c2b 16384"}; do
    set -- $cp
    PFT_LIB=$lib timeout 200 python bench.py --config $1 --p $2 --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print('$lib'.split('/')[-1], '$1', $2, 'r', d['config']['r'], 'us', round(d['ms_per_step']*1e3,2), 'GB/s', round(d['input_gbs']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/ab_tc.log 2>&1
  done
done
done
for p in 256 512; do PFT_LIB=tools/_variants/lib_tl.so timeout 120 python tools/timeline_c3.py $p 4096 >> $O/tl_c3_tc.log 2>&1; done
