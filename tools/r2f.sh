O=gpurun_out
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $O/pt_gpu.log 2>&1; tail -60 $O/pt_gpu.log
