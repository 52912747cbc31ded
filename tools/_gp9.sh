python -m pytest tests/test_gpu_parity.py -q -x -k "gmres" > gpurun_out/t9.log 2>&1; echo "parity rc=$?"; tail -c 300 gpurun_out/t9.log
for dl in 1 0; do AIRG_DEVLOOP=$dl python tools/gm_probe.py --fast 1; done
