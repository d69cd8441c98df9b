#!/usr/bin/env bash
# Lloyd iteration loop on the GPU box: parity tests, stats/timeline probe, bench.  usage: bash tools/lloyd_session.sh TAG
# (the probes need a probe build: python tools/ab_build.py probes 'KT_LLOYD_PROBES 0=>KT_LLOYD_PROBES 1')
T=gpurun_out/$1; mkdir -p $T
timeout 700 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $T/tests.log 2>&1; echo tests rc=$?; tail -3 $T/tests.log
KT_LIB_PATH=build/ab/probes.so KT_LLOYD_STATS=1 python tools/lloyd_probe.py > $T/stats.txt 2>&1
KT_LIB_PATH=build/ab/probes.so KT_LLOYD_TIMELINE=1 python tools/lloyd_probe.py > $T/timeline.txt 2>&1
python bench.py --no-cpu-baseline > $T/bench.json 2>$T/bench.err; cut -c1-200 $T/bench.json
grep "rep 2" $T/stats.txt
