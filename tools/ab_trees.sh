#!/usr/bin/env bash
# A/B of K2 variants built by tools/ab_build.py: bash tools/ab_trees.sh TAG v1 v2 ...
T=gpurun_out/$1; shift; mkdir -p $T
for round in 1 2; do
  for v in "$@"; do
    echo "$v $(KT_LIB_PATH=build/ab/$v.so timeout 120 python tools/trees_probe.py 2>&1 | tail -1)" | tee -a $T/ab.txt
  done
done
