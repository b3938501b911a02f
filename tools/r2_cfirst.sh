O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_cf.log 2>&1; echo "rc=$?" >> $O/pytest_cf.log
timeout 300 python tools/sweep.py spx1e6_u01 spx1e6_n01 spx1e6_u01_tight spx1e6_n01_tight spx1e6_u01_formula spx l1 > $O/sweep_cf.log 2>&1
CQK_SPX_CAPTURE=0 timeout 300 python tools/sweep.py spx1e6_u01 spx1e6_n01 spx1e6_u01_tight spx1e6_n01_tight spx1e6_u01_formula > $O/sweep_cf0.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py spx_n01 1e6 > $O/tl_c1n_cf.log 2>&1
