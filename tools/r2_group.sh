O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x > $O/pytest_group.log 2>&1; echo "rc=$?" >> $O/pytest_group.log
for t in racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_$t.log 2>&1; echo "rc=$?" >> $O/sanitize_$t.log
done
CQK_DEVICES=0,0 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_racecheck_group.log 2>&1; echo "rc=$?" >> $O/sanitize_racecheck_group.log
