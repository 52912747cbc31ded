#!/bin/bash
# Round-2 profiles of the C4 headline solve (fast mode, device GMRES kernels
# launched one by one so ncu sees them). Plain runs first, ncu after.
set -u
mkdir -p gpurun_out
python tools/profile_solve.py --config 4 --what solve > gpurun_out/p2_plain.log 2>&1 || { echo "plain solve failed"; cat gpurun_out/p2_plain.log; exit 1; }
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r2_c4_solve_launches.csv \
    python tools/profile_solve.py --config 4 --what solve > gpurun_out/p2_ncu_launch.log 2>&1; echo "launch list rc=$?"
# --set full: level-0 restriction (first rows_lanes of the solve), level-0 x-update
# (19th k_fused_x), the GMRES A z (EpiGmSpmv), the Gram sweep (k_gm_sweep<3>, 16th)
for spec in "r0:rows_lanes:0" "fusedx0:k_fused_x:18" "gmspmv:EpiGmSpmv:5" "sweep3:k_gm_sweep:31"; do
  IFS=: read name kre skip <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k "regex:$kre" --launch-skip "$skip" -c 1 -o "gpurun_out/r2_${name}_full" -f \
      python tools/profile_solve.py --config 4 --what solve > "gpurun_out/p2_${name}.log" 2>&1; echo "$name rc=$?"
done
