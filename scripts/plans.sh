# world-1 step schedules (bench.py --plan), with and without DBP_OPT_OVERLAP_PREV
for p in "admm_ul,admm_dl,cg_ul" "admm_ul,cg_ul,admm_dl" "cg_ul,admm_ul,admm_dl" "admm_dl,admm_ul,cg_ul" "admm_ul,admm_dl|cg_ul" "admm_ul,cg_ul|admm_dl"; do
  for o in "" "--no-overlap"; do
  python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-table2 --no-configs --e2e-steps 1 --plan "$p" $o 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p', '$o', round(d['value'],4), round(d['ms_per_step']*1000,1))"
  done
done
