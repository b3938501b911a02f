O=gpurun_out; mkdir -p $O
for f in 12 28; do
  CQK_TMA_FLAGS=$f timeout 300 python tools/sweep.py spx l1 spx_formula rows > $O/sweep_split_$f.log 2>&1
  CQK_TMA_FLAGS=$f CQK_SPX_CAPTURE=0 timeout 300 python tools/sweep.py spx l1 > $O/sweep_split_nc_$f.log 2>&1
done
