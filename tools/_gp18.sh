python -m pytest tests/ -q -x -m gpu > gpurun_out/t18.log 2>&1; echo "gpu suite rc=$?"; tail -c 400 gpurun_out/t18.log
python bench.py --steps 10 --warmup 3 > gpurun_out/b18.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/b18.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['iterations'], d['setup_ms'], d['roofline']['frac'], d['roofline']['traffic'], d['gpu_launches'], d['e2e']['value'], d['other_mode']['value'], {k:(v.get('value'), v.get('setup_ms')) for k,v in d['configs'].items()}, d['cf_split_ms'], d['cpu_baseline']['value'])"
