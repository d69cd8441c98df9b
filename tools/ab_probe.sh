#!/usr/bin/env bash
# A/B of engine variants on the knee-scan probe, printing the chosen kernels' times:
#   bash tools/ab_probe.sh TAG 'kernel1|kernel2' v1 v2 ...
T=gpurun_out/$1; K=$2; shift 2; mkdir -p $T
for round in 1 2; do
  for v in "$@"; do
    echo "$v $(KT_LIB_PATH=build/ab/$v.so timeout 120 python tools/lloyd_probe.py 2>&1 | grep 'rep 2' | grep -oE "'($K)': [0-9.]*" | tr '\n' ' ')" | tee -a $T/ab.txt
  done
done
