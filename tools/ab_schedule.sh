O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_bench_plans.py -x -q -k "c2b or c4 or overlap or batch3 or consumes" > $O/ab1_pytest.log 2>&1; echo "exit $?" >> $O/ab1_pytest.log
timeout 900 python tools/quick_time.py c2b c4 c1 c2a c2c --variant schedule=static --variant schedule=auto > $O/ab1_time.log 2>&1
timeout 600 python tools/quick_time.py c3 --variant schedule=static --variant schedule=auto >> $O/ab1_time.log 2>&1
