# Round-2 closing measurement at HEAD: bench (both arms), the bench command's launch list, ncu --set full of the
# step's three kernels.  Summaries: LAUNCH_CMD=... python scripts/make_profiles.py r02 gpurun_out/r02_launches.csv ...
set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-table2 --no-configs > gpurun_out/r02_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused --launch-skip 1 --launch-count 1 -o gpurun_out/r02_full_bf python scripts/prof_solver.py --solver bf --config D --reps 2 > gpurun_out/r02_full_bf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused --launch-skip 1 --launch-count 1 -o gpurun_out/r02_full_admm python scripts/prof_solver.py --solver admm --config C --reps 2 > gpurun_out/r02_full_admm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cg_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02_full_cg python scripts/prof_solver.py --solver cg --config C --reps 2 > gpurun_out/r02_full_cg.log 2>&1
ls -la gpurun_out/ | tail -12
