O=gpurun_out
for f in 0 1; do
  if [ $f = 0 ]; then export CQK_FUSED_MIN_N=1000000000000; else unset CQK_FUSED_MIN_N; fi
  CQK_TIMELINE=1 timeout 300 python tools/timeline.py weak > $O/tl_f$f.log 2>&1; echo "fused=$f"; cut -c1-130 $O/tl_f$f.log | tail -11
done
unset CQK_FUSED_MIN_N
timeout 300 python tools/sweep.py weak corr unc8 jac unc7 weak7 > $O/sweep_f1.log 2>&1; cut -c1-200 $O/sweep_f1.log
