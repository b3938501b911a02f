for f in 1e18 0; do for g in 60 148; do
DIAG_FUSED_MIN=$f CQK_TIMELINE=1 timeout 60 python tools/diag_sharded.py $g 600011 0 2>&1 | tail -3
done; done
