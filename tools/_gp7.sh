mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "gmres or p5 or realloc" > gpurun_out/t7.log 2>&1; echo "parity rc=$?"; tail -c 800 gpurun_out/t7.log
python -m pytest tests/test_gpu_layouts.py -q -x -k "fast" > gpurun_out/t7b.log 2>&1; echo "fast rc=$?"; tail -c 800 gpurun_out/t7b.log
python -m pytest tests/test_gpu_fullsize.py -q -x -k "C4" > gpurun_out/t7c.log 2>&1; echo "full C4 rc=$?"; tail -c 1500 gpurun_out/t7c.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/b7.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/b7.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['iterations'], d['setup_ms'], d['roofline']['frac'], d['gpu_launches'], d['other_mode'])"
tail -5 gpurun_out/b7.log | cut -c1-600
