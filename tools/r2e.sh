O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pt_gpu.log 2>&1; tail -15 $O/pt_gpu.log
python tools/replay_reference_tests.py run > $O/refsuite.log 2>&1; tail -3 $O/refsuite.log
CQK_BENCH_DEVICE=0 timeout 300 python bench.py --gpus 2 --size 2000000 --steps 3 --warmup 3 > $O/b_n2_c3.log 2>&1; tail -c 1500 $O/b_n2_c3.log
timeout 300 python bench.py --steps 10 --warmup 3 > $O/b_c3.log 2>&1; tail -c 3000 $O/b_c3.log
