O=gpurun_out; mkdir -p $O
CQK_TIMELINE=1 timeout 300 python tools/timeline.py spx_u01 1e6 > $O/tl_c1u.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py spx_n01 1e6 > $O/tl_c1n.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py unc 1e7 > $O/tl_c2.log 2>&1
CQK_TIMELINE=1 timeout 300 python tools/timeline.py l1_n01 1e8 > $O/tl_l18.log 2>&1
