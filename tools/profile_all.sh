# Round evidence: bench lines, the bench launch list and ncu --set full
# captures of the three hot kernels.  Usage: bash tools/profile_all.sh r01
R=${1:-r01}
O=gpurun_out
python bench.py > $O/bench_$R.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$R.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $O/ncu_launch_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cqk_tma -s 2 -c 1 \
    -o $O/prof_solve_$R python tools/profile_solve.py --reps 3 > $O/ncu_solve_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spx_tma -s 2 -c 1 \
    -o $O/prof_spx_$R python tools/profile_solve.py --kind simplex --reps 3 > $O/ncu_spx_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spx_rows -s 2 -c 1 \
    -o $O/prof_rows_$R python tools/profile_solve.py --kind rows --n 268435456 --reps 3 > $O/ncu_rows_$R.log 2>&1
