# A/B the TMA engine configurations (tile, stages, consumer warps) on timelines
for v in ${VARIANTS:-1920_2_15 960_4_15 1536_3_12}; do
  export CQK_LIB=paper_2603_15910_b200/lib/variants/lib_$v.so
  echo "== $v" >> gpurun_out/variants.txt
  timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1 >> gpurun_out/variants.txt
  for k in weak jac corr; do timeout 120 python tools/timeline.py $k 2>&1 | cut -c1-100 >> gpurun_out/variants.txt; done
  timeout 120 python tools/timeline.py unc 1e7 2>&1 | cut -c1-100 >> gpurun_out/variants.txt
done
