#!/usr/bin/env bash
# A/B of the headline bench under env settings: bash tools/ab_e2e.sh TAG 'ENV=..' 'ENV=..' ...
T=gpurun_out/$1; shift; mkdir -p $T
for round in 1 2; do
  for v in "$@"; do
    env $v python bench.py --no-cpu-baseline --no-wall95 --no-extra-configs > $T/b.json 2> $T/b.err
    python - "$v" $T/b.json <<'PY' | tee -a $T/ab.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().splitlines()[-1])
print(sys.argv[1], "value %.4g e2e %.4g ms/step %.4f lloyd %.4f parity %s" % (d["value"], d["e2e"]["value"], d["ms_per_step"], d["kernels"]["lloyd"]["ms_per_step"], d["parity"]["ok"]))
PY
  done
done
