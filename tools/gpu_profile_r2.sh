#!/bin/bash
# Round-2 profiles of the C4 headline solve (fast mode, device GMRES kernels
# launched one by one so ncu sees them). Plain runs first, ncu after.
set -u
mkdir -p gpurun_out
python tools/profile_solve.py --config 4 --what solve > gpurun_out/p2_plain.log 2>&1 || { echo "plain solve failed"; cat gpurun_out/p2_plain.log; exit 1; }
python tools/profile_solve.py --config 4 --what spmv > gpurun_out/p2_plain_spmv.log 2>&1 || { echo "plain spmv failed"; exit 1; }
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r2_c4_solve_launches.csv \
    python tools/profile_solve.py --config 4 --what solve > gpurun_out/p2_ncu_launch.log 2>&1; echo "launch list rc=$?"
for spec in "spmv0:rows_lanes:0:spmv" "fusedx:k_fused_x:60:solve" "sweep1:k_gm_sweep:31:solve" "fres:rows_lanes:81:solve"; do
  IFS=: read name kre skip what <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k "regex:$kre" --launch-skip "$skip" -c 1 -o "gpurun_out/r2_${name}_full" -f \
      python tools/profile_solve.py --config 4 --what $what > "gpurun_out/p2_${name}.log" 2>&1; echo "$name rc=$?"
done
