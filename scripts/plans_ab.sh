# A/B of the two best world-1 schedules, alternated
for rep in 1 2 3; do
  for cfg in "admm_ul,admm_dl,cg_ul|" "admm_ul,admm_dl|cg_ul|--no-overlap"; do
    p="${cfg%|*}"; o="${cfg##*|}"; [ "$p" = "admm_ul,admm_dl" ] && p="admm_ul,admm_dl|cg_ul"
    python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-table2 --no-configs --e2e-steps 1 --plan "$p" $o 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p', '$o', round(d['value'],4), round(d['ms_per_step']*1000,2))"
  done
done
