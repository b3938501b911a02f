O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_golden.py tests/test_gpu_degenerate.py tests/test_gpu_sharded.py tests/test_gpu_group.py tests/test_gpu_parity.py -q -x > $O/pytest_fg.log 2>&1; echo "rc=$?" >> $O/pytest_fg.log
CQK_TIMELINE=1 timeout 300 python tools/timeline.py weak > $O/tl_weak_g1.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py unc 1e7 > $O/tl_unc7_g1.log 2>&1
for cr in 0.5 0.4 0.3; do
  CQK_COMPACT_RATIO=$cr timeout 600 python tools/sweep.py weak corr unc8 unc7 weak7 > $O/sweep_g1_cr$cr.log 2>&1
done
CQK_FUSED_GUESS=0 timeout 600 python tools/sweep.py weak corr unc8 unc7 weak7 > $O/sweep_g0.log 2>&1
