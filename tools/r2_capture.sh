O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_capture.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_gridstep.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_api.py tests/test_gpu_alg2.py -q > $O/pytest_cap.log 2>&1; echo "rc=$?" >> $O/pytest_cap.log
timeout 600 python tools/sweep.py spx l1 spx_formula spx1e6_u01 spx1e6_n01 > $O/sweep_cap.log 2>&1
CQK_SPX_CAPTURE=0 timeout 600 python tools/sweep.py spx l1 spx_formula > $O/sweep_nocap.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py l1 > $O/tl_l1_cap.log 2>&1
timeout 600 python tools/c4_l1.py > $O/c4_cap.log 2>&1
