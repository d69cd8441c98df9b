#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over small fixtures of every
# kernel family (K2 trees, K3 landscape, K6 dedup, K7 init, K8 Lloyd resident + streaming +
# reseed, knee, K9 mode, K10 SA, K1/K4/K5 RL round + tcgen05 GEMMs, top-k, report, sharded
# Lloyd).  usage (GPU box): bash tools/sanitize.sh TAG [tools...]
T=gpurun_out/$1; shift; mkdir -p $T
TOOLS=${*:-"memcheck racecheck synccheck initcheck"}
SEL='test_predict_bit_exact_vs_reference or test_landscape_vs_reference or test_kmeans_vs_reference or test_knee_vs_reference or test_adaptive_sample_vs_reference or (test_lloyd_variants_vs_oracle and 0) or test_sa_vs_reference or test_first_round_matches_reference or test_top_unvisited_vs_reference or test_report_vs_reference or test_gpu_sharded_reseed_vs_oracle or test_gemm'
FILES="tests/test_gpu_parity.py tests/test_gpu_rl.py tests/test_gpu_tune.py tests/test_gpu_report.py tests/test_gpu_shard.py tests/test_gpu_gemm.py"
for tool in $TOOLS; do
  extra=""
  sel=$SEL
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  [ $tool = memcheck ] && extra="--leak-check no"
  # racecheck / synccheck abort kernels that use cp.async.bulk + mbarrier (K1 rollout) or
  # tcgen05 (K5 GEMMs) with "unspecified launch failure"; memcheck / initcheck cover those
  if [ $tool = racecheck ] || [ $tool = synccheck ]; then sel="($SEL) and not test_first_round and not test_gemm"; fi
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 200 \
    python -m pytest $FILES -m gpu -q -x -p no:cacheprovider -k "$sel" > $T/san_$tool.txt 2>&1
  rc=$?
  grep -h "hazard detected\|Read Thread\|Write Thread\|^=========     at " $T/san_$tool.txt | sed 's/block ([0-9,]*)//; s/__shared__ 0x[0-9a-f]*//; s/Thread ([0-9,]*)//; s/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -20 > $T/san_${tool}_sites.txt
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $T/san_$tool.txt | tail -3 | tr '\n' ' ')"
done
