#!/bin/bash
# A/B of the solve row kernels (default CSR thread-per-row, pipelined batches).
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_default.log 2>&1
AIRG_PDL=0 timeout 300 python tools/trace_solve.py --out gpurun_out/trace_default_nopdl.txt > /dev/null 2>&1
