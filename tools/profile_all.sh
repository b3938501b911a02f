# Round evidence: bench lines, the bench launch list and ncu --set full
# captures of the three hot kernels.  Usage: bash tools/profile_all.sh r02
R=${1:-r02}
O=gpurun_out
mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:cqk_tma -s 2 -c 1 \
    -o $O/prof_solve_$R -f python tools/profile_solve.py --reps 3 > $O/ncu_solve_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spx_tma -s 2 -c 1 \
    -o $O/prof_spx_$R -f python tools/profile_solve.py --kind simplex --reps 3 > $O/ncu_spx_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spx_rows -s 2 -c 1 \
    -o $O/prof_rows_$R -f python tools/profile_solve.py --kind rows --n 268435456 --reps 3 > $O/ncu_rows_$R.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv \
    python bench.py --steps 6 --warmup 3 --no-cpu --e2e-steps 0 > $O/ncu_launch_$R.log 2>&1
python bench.py > $O/bench_$R.log 2>&1
python bench.py --impl reference > $O/bench_ref_$R.log 2>&1
# summaries on the box; only the solve report travels back (gpurun_out <= 64 MiB)
mkdir -p $O/profiles_box
python tools/make_profiles.py $R $O/profiles_box > /dev/null 2>&1
rm -f $O/prof_spx_$R.ncu-rep $O/prof_rows_$R.ncu-rep
