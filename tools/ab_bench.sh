# A/B of two library builds on the bench's rebuild / solve times (2 steps each, twice)
for v in old new old new; do
  AMGR_LIB=abtest/lib_$v.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-strategies 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), 'rebuild', round(d['rebuild_ms_per_step'],3), 'solve', round(d['solve_ms_per_step'],2), d['iterations'])"
done
