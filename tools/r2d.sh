O=gpurun_out
CQK_BENCH_DEVICE=0 timeout 300 python bench.py --gpus 2 --size 2000000 --steps 3 --warmup 3 > $O/b_n2_c3.log 2>&1; tail -c 2500 $O/b_n2_c3.log
CQK_BENCH_DEVICE=0 timeout 300 python bench.py --gpus 2 --config c4 --size 20000000 --steps 3 --warmup 3 > $O/b_n2_c4.log 2>&1; tail -c 1500 $O/b_n2_c4.log
CQK_BENCH_DEVICE=0 timeout 300 python bench.py --gpus 2 --config c5 --size 4096 --steps 3 --warmup 3 > $O/b_n2_c5.log 2>&1; tail -c 1500 $O/b_n2_c5.log
python tools/replay_reference_tests.py run > $O/refsuite.log 2>&1; tail -3 $O/refsuite.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > $O/pt_full.log 2>&1; tail -15 $O/pt_full.log
