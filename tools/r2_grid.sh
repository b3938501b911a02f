O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_gridstep.py tests/test_gpu_sharded.py tests/test_gpu_fused.py tests/test_gpu_multi.py tests/test_gpu_group.py tests/test_gpu_parity.py tests/test_gpu_golden.py -q > $O/pytest_grid.log 2>&1; echo "rc=$?" >> $O/pytest_grid.log
timeout 600 python tools/sweep.py unc7 weak7 spx1e6_u01 spx1e6_n01 weak corr spx > $O/sweep_grid.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py unc 1e7 > $O/tl_unc7_grid.log 2>&1
timeout 900 python tools/replay_reference_tests.py run > $O/refsuite.log 2>&1
