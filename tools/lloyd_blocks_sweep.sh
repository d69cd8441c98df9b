#!/usr/bin/env bash
# Resident-Lloyd grid size vs the tuning loop's small point sets (wall-to-95 rounds).
# usage: bash tools/lloyd_blocks_sweep.sh OUTDIR [blocks...]
OUT=${1:-gpurun_out/blocks}; shift || true
mkdir -p "$OUT"
for b in ${*:-148 96 64 48 32 24 16 8 4}; do
  KT_LLOYD_BLOCKS=$b timeout 300 python tools/w95_probe.py > "$OUT/w95_b$b.txt" 2>&1
  echo "blocks=$b $(grep -m1 'sync=False' "$OUT/w95_b$b.txt") $(grep ' lloyd ' "$OUT/w95_b$b.txt")"
done
