O=gpurun_out
mkdir -p $O
for f in 0 1; do
  if [ $f = 0 ]; then export CQK_FUSED_MIN_N=1000000000000; else unset CQK_FUSED_MIN_N; fi
  timeout 300 python tools/sweep.py weak corr unc8 jac unc7 weak7 > $O/sweep_f$f.log 2>&1; echo "fused=$f"; cat $O/sweep_f$f.log | tail -8
done
unset CQK_FUSED_MIN_N
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pt_gpu.log 2>&1; tail -15 $O/pt_gpu.log
