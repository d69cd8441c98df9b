#!/usr/bin/env bash
# RL bench (configs[1]) A/B: bash tools/ab_rl30.sh TAG 'ENV=..' ...  (KT_LIB_PATH=build/ab/x.so selects a variant)
T=gpurun_out/$1; shift; mkdir -p $T
for round in 1 2; do
  for v in "$@"; do
    env $v timeout 600 python bench.py --workload rl > $T/rl.json 2> $T/rl.err
    python - "$v" $T/rl.json <<'PY' | tee -a $T/ab_rl.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().splitlines()[-1])
k = d.get("kernels", {})
print(sys.argv[1], "ms/step %.2f lloyd %.3f kernels %.2f" % (d["ms_per_step"], k.get("lloyd", {}).get("ms", 0), sum(x["ms"] for x in k.values())))
PY
  done
done
