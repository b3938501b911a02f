O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_capture.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_gridstep.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_api.py tests/test_gpu_spg.py -q > $O/pytest_sp.log 2>&1; echo "rc=$?" >> $O/pytest_sp.log
timeout 600 python tools/sweep.py spx l1 > $O/sweep_sp.log 2>&1
timeout 600 python tools/c4_l1.py > $O/c4_sp.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py l1_n01 1e8 > $O/tl_l18_sp.log 2>&1
