#!/bin/bash
# A/B of engine builds / runtime knobs on the C2 solve: per-iteration cost
# (tools/iter_cost.py), interleaved twice.
#   tools/ab_variants.sh [spec ...]   spec = <tag> (variants/libairg_<tag>.so)
#                                     or <tag>+VAR=val[,VAR=val] (lib + env; tag "base" = in-tree lib)
#   -> gpurun_out/ab_variants.txt
set -u
mkdir -p gpurun_out
out=gpurun_out/ab_variants.txt
: > $out
specs=("$@")
[ ${#specs[@]} -eq 0 ] && specs=($(ls paper_2408_08262_b200/variants/ | sed -n 's/^libairg_\(.*\)\.so$/\1/p'))
run() {  # tag envlist
  local lib=""
  [ "$1" != base ] && lib=$PWD/paper_2408_08262_b200/variants/libairg_$1.so
  ( [ -n "$lib" ] && export AIRG_LIB=$lib
    IFS=, ; for kv in $2; do [ -n "$kv" ] && export "$kv"; done
    timeout 300 python ${AB_CMD:-tools/iter_cost.py} ) >> $out 2>&1
}
for rep in 1 2; do
  echo "== base" >> $out; run base ""
  for s in "${specs[@]}"; do
    tag=${s%%+*}; envs=""; [ "$tag" != "$s" ] && envs=${s#*+}
    echo "== $s" >> $out; run "$tag" "$envs"
  done
done
cat $out
