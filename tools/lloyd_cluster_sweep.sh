#!/usr/bin/env bash
# One-cluster Lloyd launch vs the cooperative grid at small point counts.
# usage: bash tools/lloyd_cluster_sweep.sh OUTDIR
OUT=${1:-gpurun_out/cluster}; mkdir -p "$OUT"
for c in 0 16 8 4; do
  for n in 1000 5000 20000 65536; do
    echo "cluster=$c n=$n $(KT_LLOYD_CLUSTER=$c timeout 120 python tools/lloyd_probe.py $n 2>&1 | grep 'rep 2' | grep -oE "passes=[0-9]+|'lloyd': [0-9.]*" | tr '\n' ' ')"
  done
  echo "cluster=$c w95 $(KT_LLOYD_CLUSTER=$c timeout 300 python tools/w95_probe.py 2>&1 | grep -m1 'sync=False') $(KT_LLOYD_CLUSTER=$c timeout 300 python tools/w95_probe.py 2>&1 | grep ' lloyd ')"
done 2>&1 | tee "$OUT/sweep.txt"
