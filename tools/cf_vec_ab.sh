# A/B of the CF split variants on C2 (cf_split_ms, per-level-sync ms, setup ms)
for cfg in "AIRG_CF_SMALL=0" "AIRG_CF_SMALL=30000" "AIRG_CF_SMALL=70000" "AIRG_CF_SMALL=131072" "AIRG_CF_SMALL=300000" "AIRG_CF_SMALL=800000"; do
  echo "$cfg"; env $cfg python bench.py --steps 3 --warmup 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['cf_split_ms'], d['cf_split_ms_sync_each_level'], d['setup_ms'])"
done
