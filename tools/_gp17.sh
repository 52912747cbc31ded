python -m pytest tests/test_gpu_parity.py tests/test_gpu_layouts.py -q -x -k "gmres or fast" > gpurun_out/t17.log 2>&1; echo "tests rc=$?"; tail -c 200 gpurun_out/t17.log
python tools/gm_probe.py --fast 1
