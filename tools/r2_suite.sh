O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python tools/sweep.py spx l1 spx1e6_u01 spx1e6_n01 > $O/sweep_cap.log 2>&1
timeout 600 python tools/c4_l1.py > $O/c4_cap.log 2>&1
