#!/usr/bin/env bash
# ncu --set full capture of one kernel from a short bench run: tools/prof.sh <kernel-regex> <tag> [bench args]
K=$1; TAG=$2; shift 2
mkdir -p gpurun_out/$TAG
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/$TAG/prof_$K \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-wall95 "$@" > gpurun_out/$TAG/prof_$K.log 2>&1
echo "prof $K rc=$?"
