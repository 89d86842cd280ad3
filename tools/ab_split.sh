O=gpurun_out; mkdir -p $O; L=$O/ab_split.log; : > $L
q() { echo "## $C $V" >> $L; timeout 300 python tools/quick_time.py $C --reps 100 --variant "$V" >> $L 2>&1; }
for C in c2b c4 c1 c2a c2c; do
  for V in "split=0" "split=1"; do q; done
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py -x -q > $O/ab_split_pytest.log 2>&1; echo "exit $?" >> $O/ab_split_pytest.log
