# A/B of the SpGEMM finish (rank placement vs bitonic network) on the C2 setup
for cfg in "AIRG_SPGEMM_SORT=bitonic" "AIRG_SPGEMM_SORT=rank"; do
  echo "$cfg"; env $cfg python bench.py --steps 3 --warmup 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('setup_ms', d['setup_ms'], 'solve ms', d['ms_per_step'])"
done
