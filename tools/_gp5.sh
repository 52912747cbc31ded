mkdir -p gpurun_out
python -m pytest tests/test_gpu_layouts.py -q -x > gpurun_out/t5.log 2>&1; echo "tests rc=$?"
tail -c 1500 gpurun_out/t5.log
python tools/trace_solve.py --config 4 --max-its 8 --fast 1 --out gpurun_out/c4_rich_fused.txt > gpurun_out/tr5.log 2>&1
head -25 gpurun_out/c4_rich_fused.txt; tail -5 gpurun_out/tr5.log
python tools/trace_solve.py --config 4 --outer 1 --fast 1 --out gpurun_out/c4_gmres_fused.txt > /dev/null 2>&1
head -30 gpurun_out/c4_gmres_fused.txt
