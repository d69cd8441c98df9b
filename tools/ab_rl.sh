#!/usr/bin/env bash
# RL-step A/B of engine variants: bash tools/ab_rl.sh TAG v1 v2 ...
T=gpurun_out/$1; shift; mkdir -p $T
for v in "$@"; do
  KT_LIB_PATH=build/ab/$v.so timeout 300 python bench.py --workload rl --no-cpu-baseline --steps 5 > $T/rl_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('$T/rl_$v.json')); k=d['kernels']
print('$v', round(d['ms_per_step'], 2), 'gemm ms', round(d['roofline']['gemm_ms_per_step'], 2), {n: k[n]['ms'] for n in ('tc_gemm_wgrad', 'reduce_splits') if n in k})"
done
