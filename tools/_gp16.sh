python -m pytest tests/test_ops.py tests/test_gpu_layouts.py tests/test_kats.py -q -x -k "cf or split or fused or kat" > gpurun_out/t16.log 2>&1; echo "tests rc=$?"; tail -c 300 gpurun_out/t16.log
python -m pytest tests/test_gpu_parity.py -q -x -k "p1 or p2" > gpurun_out/t16b.log 2>&1; echo "p1p2 rc=$?"; tail -c 300 gpurun_out/t16b.log
python tools/cf_batch_time.py 2; python tools/cf_batch_time.py 4
