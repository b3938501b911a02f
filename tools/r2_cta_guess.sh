O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_golden.py tests/test_gpu_degenerate.py tests/test_gpu_sharded.py tests/test_gpu_group.py tests/test_gpu_fullsize.py tests/test_gpu_gridstep.py -q > $O/pytest_cg.log 2>&1; echo "rc=$?" >> $O/pytest_cg.log
timeout 1500 python tools/fused_ab.py 1e7,1e8 > $O/fused_ab_cg.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py weak > $O/tl_weak_cg.log 2>&1
