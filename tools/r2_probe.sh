# Round-2 probes: per-pass timelines, size sweep, reference-suite replay, sanitizers.
O=gpurun_out; mkdir -p $O
for k in weak corr; do CQK_TIMELINE=1 timeout 300 python tools/timeline.py $k > $O/tl_$k.log 2>&1; done
CQK_TIMELINE=1 timeout 300 python tools/timeline.py unc 1e7 > $O/tl_unc7.log 2>&1
timeout 600 python tools/sweep.py weak corr unc8 jac unc7 weak7 > $O/sweep.log 2>&1
timeout 900 python tools/replay_reference_tests.py run > $O/refsuite.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_$t.log 2>&1; echo "rc=$?" >> $O/sanitize_$t.log
done
