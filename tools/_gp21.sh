python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
python -m pytest tests/ -q -m gpu > gpurun_out/t21.log 2>&1; echo "gpu suite rc=$?"; tail -c 600 gpurun_out/t21.log
