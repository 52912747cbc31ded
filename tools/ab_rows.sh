#!/bin/bash
# A/B of the row decompositions (tiled.cuh) on the C2 solve: default, forced
# thread-per-row, forced warp tiles.
for mode in "" thread tiles; do
  AIRG_ROWS=$mode timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${mode:-auto}.log 2>&1
done
