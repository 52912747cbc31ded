AIRG_GM_FLAT=1 python tools/gm_probe.py --fast 1 2>&1 | tail -3
AIRG_GM_FLAT=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/gm_launches.csv python tools/gm_probe.py --fast 1 --profile > gpurun_out/gm_ncu.log 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/gm_launches.csv | head -30
