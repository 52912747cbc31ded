#!/bin/bash
# Round-2 profiles of the C4 headline solve (fast mode; the device GMRES
# kernels launched one by one so ncu sees them: AIRG_GM_FLAT=1 in
# tools/profile_solve.py). Plain runs first, ncu after; summaries by
# tools/profile_c4.py into profiles/.
set -u
mkdir -p gpurun_out
python tools/profile_solve.py --config 4 --what solve > gpurun_out/p2_plain.log 2>&1 || { echo "plain solve failed"; cat gpurun_out/p2_plain.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/r2_c4_solve_launches.csv \
    python tools/profile_solve.py --config 4 --what solve > gpurun_out/p2_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/r2_c4_spmv.csv \
    python tools/profile_solve.py --config 4 --what spmv > gpurun_out/p2_spmv.log 2>&1; echo "spmv rc=$?"
CF_CONFIG=4 python tools/ncu_cf.py > gpurun_out/p2_cf_plain.log 2>&1 && \
CF_CONFIG=4 timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/r2_c4_cf.csv \
    python tools/ncu_cf.py > gpurun_out/p2_cf.log 2>&1; echo "cf rc=$?"
# --set full: level-0 descent [R; W E_F^T] b (EpiStore2), level-0 one-pass
# x-update (19th k_fused_x), a level-4 x-update (15th), a late Gram sweep
for spec in "desc0:EpiStore2:0" "fusedx0:k_fused_x:18" "fusedx4:k_fused_x:14" "sweep:k_gm_sweep:31"; do
  IFS=: read name kre skip <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      --kernel-name-base demangled -k "regex:$kre" --launch-skip "$skip" -c 1 -o "gpurun_out/r2_${name}_full" -f \
      python tools/profile_solve.py --config 4 --what solve > "gpurun_out/p2_${name}.log" 2>&1; echo "$name rc=$?"
done
