#!/bin/bash
# The bounds-checked library (build.py --checked: every computed workspace / output / input index
# checked, a violation traps) over every device form and the GPU parity suites.
O=gpurun_out; mkdir -p $O
export PFT_LIB=$PWD/paper_2008_12559_b200/libpft_b200_checked.so
timeout 900 python tools/sanitize.py > $O/checked_sanitize.log 2>&1; echo "exit $?" >> $O/checked_sanitize.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py tests/test_pft2d.py tests/test_gpu_sharded.py tests/test_signal_io.py -m gpu -q > $O/checked_pytest.log 2>&1; echo "exit $?" >> $O/checked_pytest.log
unset PFT_LIB
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_checked_run.log 2>&1; echo "exit $?" >> $O/pytest_gpu_checked_run.log
