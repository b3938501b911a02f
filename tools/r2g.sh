O=gpurun_out
mkdir -p $O
python tools/rows_ab.py > $O/rows_ab.log 2>&1; tail -3 $O/rows_ab.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "rows or c5 or sharpened" > $O/pt_rows.log 2>&1; tail -15 $O/pt_rows.log
