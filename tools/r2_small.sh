O=gpurun_out; mkdir -p $O
for m in 4000000 100000; do
  CQK_SPX_CAPTURE_MIN_N=$m timeout 300 python tools/sweep.py spx1e6_u01 spx1e6_n01 spx1e6_u01_tight spx1e6_n01_tight > $O/small_spx_$m.log 2>&1
done
for m in 4000000 500000; do
  CQK_FUSED_MIN_N=$m timeout 300 python tools/sweep.py unc6 weak6 > $O/small_cqk_$m.log 2>&1
done
