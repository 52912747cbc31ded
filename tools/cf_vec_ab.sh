# A/B of the CF split row-pass variants on C2 (cf_split_ms, per-level-sync ms, setup ms)
for cfg in "AIRG_CF_VEC=1000" "AIRG_CF_VEC=6" "AIRG_CF_VEC=3" "AIRG_CF_GROUP=4" "AIRG_CF_GROUP=8" "AIRG_CF_GROUP=16"; do
  echo "$cfg"; env $cfg python bench.py --steps 3 --warmup 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['cf_split_ms'], d['cf_split_ms_sync_each_level'], d['setup_ms'])"
done
