#!/usr/bin/env bash
# A/B of engine variants on the RL step's GEMM / colsum kernels (serial tasks, per-kernel ms per step):
#   bash tools/ab_rl.sh TAG v1 v2 ...
T=gpurun_out/$1; shift; mkdir -p $T
for v in "$@"; do
  KT_LIB_PATH=build/ab/$v.so timeout 300 python bench.py --workload rl --rl-serial --steps 5 --warmup 2 --no-cpu-baseline > $T/rl_$v.json 2> $T/rl_$v.err
  python -c "
import json;d=json.load(open('$T/rl_$v.json'));k=d['kernels']
print('$v', round(d['ms_per_step'],2), {n: k[n]['ms'] for n in k if n.startswith('tc_gemm') or n.startswith('colsum') or n=='reduce_splits'})"
done
