# per-pass timelines of the headline workloads (perf-iteration aid)
out=gpurun_out/tl_all.txt; : > $out
for k in weak corr jac; do timeout 120 python tools/timeline.py $k 2>&1 | cut -c1-110 >> $out; done
timeout 120 python tools/timeline.py unc 1e7 2>&1 | cut -c1-110 >> $out
for k in spx l1; do timeout 120 python tools/timeline.py $k 2>&1 | cut -c1-110 >> $out; done
