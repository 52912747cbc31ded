mkdir -p gpurun_out
python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/fullsize.log
