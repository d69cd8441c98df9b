#!/usr/bin/env bash
# pass-level timelines of engine variants: bash tools/ab_timeline.sh TAG v1 v2 ...
# (variants built with 'KT_LLOYD_PROBES 0=>KT_LLOYD_PROBES 1' among their replacements)
T=gpurun_out/$1; shift; mkdir -p $T
for v in "$@"; do
  KT_LIB_PATH=build/ab/$v.so KT_LLOYD_TIMELINE=1 timeout 120 python tools/lloyd_probe.py > $T/tl_$v.txt 2>&1
  echo "$v: $(python tools/timeline_sum.py $T/tl_$v.txt | sed -n 2,2p)"
  python tools/timeline_sum.py $T/tl_$v.txt | sed -n 5,7p
done
