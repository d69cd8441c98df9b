#!/usr/bin/env bash
# A/B timing of engine variants built by tools/ab_build.py: bash tools/ab_run.sh TAG v1 v2 ...
T=gpurun_out/$1; shift; mkdir -p $T
for round in 1 2; do
  for v in "$@"; do
    echo "$v $(KT_LIB_PATH=build/ab/$v.so timeout 120 python tools/lloyd_probe.py 2>&1 | grep 'rep 2' | grep -o "'lloyd': [0-9.]*")" | tee -a $T/ab.txt
  done
done
