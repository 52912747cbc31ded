python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_layouts.py tests/test_gpu_parity.py -q -x -k "fast or gmres" > gpurun_out/t19.log 2>&1; echo "tests rc=$?"; tail -c 1500 gpurun_out/t19.log
python tools/gm_probe.py --fast 1
