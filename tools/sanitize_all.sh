# compute-sanitizer over every device entry point (tools/sanitize_probe.py),
# the default routes and the large-n routes forced at probe sizes
O=gpurun_out; mkdir -p $O
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_$t.log 2>&1; echo "rc=$?" >> $O/sanitize_$t.log
  PROBE_LARGE_ROUTES=1 CQK_FUSED_MIN_N=0 CQK_SPX_CAPTURE_MIN_N=0 CQK_FUSED_GUESS=2 timeout 900 \
    compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_large_$t.log 2>&1; echo "rc=$?" >> $O/sanitize_large_$t.log
done
CQK_DEVICES=0,0 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_racecheck_group.log 2>&1; echo "rc=$?" >> $O/sanitize_racecheck_group.log
