O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_f32.py tests/test_gpu_api.py tests/test_gpu_fused.py tests/test_gpu_gridstep.py tests/test_gpu_group.py tests/test_gpu_fullsize.py -q > $O/pytest_chk.log 2>&1; echo "rc=$?" >> $O/pytest_chk.log
timeout 900 python tools/replay_reference_tests.py run > $O/refsuite.log 2>&1
