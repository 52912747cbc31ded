mkdir -p gpurun_out
python tools/fullsize_diag.py 2 > gpurun_out/diag2.log 2>&1
python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_reports.py -q -x > gpurun_out/t3.log 2>&1; echo "rc=$?"
tail -c 2500 gpurun_out/t3.log; head -30 gpurun_out/diag2.log
