#!/usr/bin/env bash
# A/B of rollout variants on the RL step (per-kernel ms per step): bash tools/ab_rollout.sh TAG v1 v2 ...
T=gpurun_out/$1; shift; mkdir -p $T
for round in 1 2; do
  for v in "$@"; do
    KT_LIB_PATH=build/ab/$v.so timeout 300 python bench.py --workload rl --steps 10 --warmup 3 --no-cpu-baseline > $T/rl_$v.json 2> $T/rl_$v.err
    python -c "
import json;d=json.loads(open('$T/rl_$v.json').read().strip().splitlines()[-1]);k=d['kernels']
print('$v', round(d['ms_per_step'],2), k['policy_rollout'])"
  done
done
