O=gpurun_out
python -m pytest tests/test_gpu_multi.py tests/test_gpu_ipc.py tests/test_gpu_sharded.py -x -q > $O/pt_multi.log 2>&1; tail -5 $O/pt_multi.log
CQK_BENCH_DEVICE=0 timeout 300 python bench.py --gpus 2 --size 2000000 --steps 3 --warmup 3 > $O/b_n2_c3.log 2>&1; tail -c 1500 $O/b_n2_c3.log
CQK_BENCH_DEVICE=0 timeout 300 python bench.py --gpus 2 --config c4 --size 20000000 --steps 3 --warmup 3 > $O/b_n2_c4.log 2>&1; tail -c 1200 $O/b_n2_c4.log
CQK_BENCH_DEVICE=0 timeout 300 python bench.py --gpus 2 --config c5 --size 4096 --steps 3 --warmup 3 > $O/b_n2_c5.log 2>&1; tail -c 1200 $O/b_n2_c5.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 > $O/b_c4.log 2>&1; tail -c 2500 $O/b_c4.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 > $O/b_c5.log 2>&1; tail -c 2500 $O/b_c5.log
timeout 600 python bench.py --config c5 --impl reference --steps 5 --warmup 1 > $O/b_c5_ref.log 2>&1; tail -c 1500 $O/b_c5_ref.log
