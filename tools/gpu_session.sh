#!/usr/bin/env bash
# One gpurun session: tests, bench, reference arm, ncu launch list + full captures.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_session.sh [tag] [what...]'
set -u
TAG=${1:-r1}; shift || true
WHAT=${*:-"tests bench ref launches full"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
for w in $WHAT; do
  case $w in
    tests)
      timeout 300 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
      timeout 900 python -m pytest tests -m gpu -q -x > "$OUT/gpu_tests.log" 2>&1; echo "gpu tests rc=$?"; tail -3 "$OUT/gpu_tests.log";;
    bench)
      timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"; cut -c1-600 "$OUT/bench.json";;
    ref)
      timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref rc=$?"; cut -c1-300 "$OUT/bench_ref.json";;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
        python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wall95 --no-extra-configs > "$OUT/launches_bench.log" 2>&1; echo "launches rc=$?";;
    full)
      for kr in lloyd:lloyd score_trees:score_trees dedup_insert:dedup_insert init_kernel:init_res_kernel; do
        k=${kr%%:*}; re=${kr#*:}
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s 2 -c 1 -o "$OUT/prof_$k" \
          python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-wall95 --no-extra-configs > "$OUT/prof_$k.log" 2>&1; echo "full $k rc=$?"
      done;;
    timeline)
      KT_LIB_PATH=build/ab/probes.so KT_LLOYD_TIMELINE=1 timeout 300 python tools/lloyd_probe.py > "$OUT/timeline.txt" 2>&1; echo "timeline rc=$?"
      python tools/timeline_sum.py "$OUT/timeline.txt" | head -4;;
    ppoerr)
      timeout 600 python tools/ppo_error.py > "$OUT/ppo_error.log" 2>&1; echo "ppoerr rc=$?"; tail -2 "$OUT/ppo_error.log";;
    rl)
      timeout 900 python bench.py --workload rl > "$OUT/bench_rl.json" 2> "$OUT/bench_rl.err"; echo "bench rl rc=$?"; cut -c1-400 "$OUT/bench_rl.json";;
    fullrl)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_rl.csv" \
        python bench.py --workload rl --steps 1 --warmup 1 --no-cpu-baseline > "$OUT/launches_rl.log" 2>&1; echo "launches rl rc=$?"
      for k in tc_gemm rollout_kernel; do
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o "$OUT/prof_$k" \
          python bench.py --workload rl --steps 1 --warmup 1 --no-cpu-baseline > "$OUT/prof_$k.log" 2>&1; echo "full $k rc=$?"
      done;;
  esac
done
