python -m pytest tests/test_gpu_layouts.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_reports.py tests/test_kats.py tests/test_ops.py -q -x > gpurun_out/t15.log 2>&1; echo "tests rc=$?"; tail -c 800 gpurun_out/t15.log
bash tools/_gp14.sh
