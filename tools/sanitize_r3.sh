#!/usr/bin/env bash
# compute-sanitizer over this session's new device paths: SA warp kernel with in-kernel start
# scoring / temperature (fused and unfused), the one-cluster Lloyd launch and small cooperative
# grids, the 256-thread tcgen05 GEMM (memcheck / initcheck only), and the device tune replays.
# usage (GPU box): bash tools/sanitize_r3.sh TAG [tools...]
T=gpurun_out/$1; shift; mkdir -p $T
TOOLS=${*:-"memcheck racecheck synccheck initcheck"}
SEL='test_sa_vs_reference or test_sa_large_vs_oracle or (test_lloyd_variants_vs_oracle and (cluster8 or grid or blocks7)) or test_kmeans_vs_reference or test_gemm_layouts or test_tune_matches_reference_driver'
FILES="tests/test_gpu_parity.py tests/test_gpu_tune.py tests/test_gpu_gemm.py"
for tool in $TOOLS; do
  extra=""
  sel=$SEL
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  [ $tool = memcheck ] && extra="--leak-check no"
  if [ $tool = racecheck ] || [ $tool = synccheck ]; then sel="($SEL) and not test_gemm"; fi
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 200 \
    python -m pytest $FILES -m gpu -q -x -p no:cacheprovider -k "$sel" > $T/san_$tool.txt 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $T/san_$tool.txt | tail -3 | tr '\n' ' ')"
done
