#!/usr/bin/env bash
# RL step time of the in-tree library vs build/ab/pre.so: bash tools/ab_rl_lib.sh TAG STEPS
T=gpurun_out/$1; S=${2:-30}; mkdir -p $T
for v in pre cur pre cur; do
  if [ $v = cur ]; then L=""; else L="KT_LIB_PATH=build/ab/pre.so"; fi
  env $L timeout 600 python bench.py --workload rl --steps $S --warmup 3 > $T/rl_$v.json 2>$T/rl_$v.err
  echo "$v $(python -c "import json;d=json.loads(open('$T/rl_$v.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), round(sum(v['ms'] for v in d['kernels'].values()),2), d['kernels']['lloyd']['ms'])")" | tee -a $T/ab.txt
done
