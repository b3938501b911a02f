# bench.py N > 1 plumbing on a one-GPU box: every rank on device 0 (CQK_BENCH_DEVICE),
# each on half the SMs (CQK_GRID_LIMIT) -- a protocol smoke test, not a number
O=gpurun_out; mkdir -p $O
export CQK_BENCH_DEVICE=0 CQK_GRID_LIMIT=74
for c in c3 c4 c5; do
  timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --config $c --e2e-steps 1 > $O/bench_n2_$c.log 2>&1; echo "rc=$?" >> $O/bench_n2_$c.log
done
