mkdir -p gpurun_out
python -m pytest tests/test_gpu_layouts.py -q -x -k "fused or fast" > gpurun_out/t6.log 2>&1; echo "tests rc=$?"
tail -c 1500 gpurun_out/t6.log
python tools/trace_solve.py --config 4 --max-its 8 --fast 1 --out gpurun_out/c4_rich_fused.txt > gpurun_out/tr6.log 2>&1
grep -A25 "^-- iter" gpurun_out/c4_rich_fused.txt; tail -3 gpurun_out/tr6.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/b6.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/b6.log
