# Evidence pass (tools/gpu_evidence.sh): GPU tests, smoke, reference-suite replay, sweep, then the profile/bench pass.
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python tools/replay_reference_tests.py run > $O/refsuite.log 2>&1
timeout 900 python tools/sweep.py weak corr unc8 jac unc7 weak7 spx l1 spx1e6_u01 spx1e6_n01 rows weak_f32 > $O/sweep.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py weak > $O/tl_weak.log 2>&1
timeout 1800 bash tools/profile_all.sh ${1:-r02}
timeout 600 python tools/c4_l1.py > $O/c4_l1.log 2>&1
