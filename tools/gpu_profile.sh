#!/bin/bash
# One GPU call: plain runs first, ncu only after they exit 0.
#   tools/gpu_profile.sh <tag>
# -> gpurun_out/<tag>_solve_launches.csv   every kernel of one C2 solve (time + DRAM bytes)
#    gpurun_out/<tag>_spmv_full.ncu-rep    --set full of the level-0 SpMV
#    gpurun_out/<tag>_fres1_full.ncu-rep   --set full of the largest F-residual launch (level 4)
set -u
tag=${1:-r1}
mkdir -p gpurun_out
python tools/profile_solve.py --what solve > gpurun_out/plain_solve.log 2>&1 || { echo "plain solve failed"; exit 1; }
python tools/profile_solve.py --what spmv > gpurun_out/plain_spmv.log 2>&1 || { echo "plain spmv failed"; exit 1; }
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${tag}_solve_launches.csv \
    python tools/profile_solve.py --what solve > gpurun_out/ncu_launch.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -c 1 \
    -o gpurun_out/${tag}_spmv_full -f python tools/profile_solve.py --what spmv \
    > gpurun_out/ncu_full.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:rows_thread_fc --launch-skip 19 -c 1 -o gpurun_out/${tag}_fres1_full -f \
    python tools/profile_solve.py --what solve > gpurun_out/ncu_fres1.log 2>&1
echo done
