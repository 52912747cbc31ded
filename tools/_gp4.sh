mkdir -p gpurun_out
python -m pytest tests/test_gpu_layouts.py tests/test_gpu_parity.py tests/test_ops.py -q -x > gpurun_out/t4.log 2>&1; echo "tests rc=$?"
tail -c 1500 gpurun_out/t4.log
python tools/trace_solve.py --config 4 --max-its 8 --out gpurun_out/c4_rich_exact.txt > /dev/null 2>&1
python tools/trace_solve.py --config 4 --max-its 8 --fast 1 --out gpurun_out/c4_rich_fast.txt > /dev/null 2>&1
head -3 gpurun_out/c4_rich_exact.txt; grep -A40 "^-- iteration" gpurun_out/c4_rich_fast.txt
