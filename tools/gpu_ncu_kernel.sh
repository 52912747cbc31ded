#!/bin/bash
# ncu --set full capture of one launch of a solve kernel (after a plain run).
#   tools/gpu_ncu_kernel.sh <out-name> <kernel-regex> <launch-skip>
set -u
mkdir -p gpurun_out
python tools/profile_solve.py --what solve > gpurun_out/plain_solve.log 2>&1 || { echo "plain solve failed"; exit 1; }
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:$2" --launch-skip "$3" -c 1 -o "gpurun_out/$1" -f \
    python tools/profile_solve.py --what solve > "gpurun_out/$1.log" 2>&1
tail -2 "gpurun_out/$1.log"
