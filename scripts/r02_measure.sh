set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-table2 --no-configs > gpurun_out/r02_ncu_bench.log 2>&1
for s in bf admm cg; do
  cfg=C; [ $s = bf ] && cfg=D
  ncu --set full --clock-control none --import-source on -k regex:k_fused --launch-skip 1 --launch-count 1 -o gpurun_out/r02_full_$s python scripts/prof_solver.py --solver $s --config $cfg --reps 2 > gpurun_out/r02_full_$s.log 2>&1
done
ls -la gpurun_out/ | tail -12
