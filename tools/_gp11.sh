python -m pytest tests/test_gpu_parity.py tests/test_gpu_layouts.py tests/test_gpu_fullsize.py tests/test_gpu_reports.py -q -x > gpurun_out/t11.log 2>&1; echo "tests rc=$?"; tail -c 600 gpurun_out/t11.log
python bench.py --steps 10 --warmup 3 > gpurun_out/b11.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/b11.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['iterations'], d['setup_ms'], d['roofline']['frac'], d['gpu_launches'], d['e2e']['value'], d['other_mode']['value'], d['configs'], d['cpu_baseline'])"
