T=gpurun_out/ab_init; mkdir -p $T
for r in 1 2; do for v in base initres; do
  echo "$v $(KT_LIB_PATH=build/ab/$v.so timeout 120 python tools/lloyd_probe.py 2>&1 | grep 'rep 2' | grep -o "'kmeanspp_init': [0-9.]*\|'lloyd': [0-9.]*" | tr '\n' ' ')" | tee -a $T/ab.txt
done; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > $T/tests.txt
KT_INIT_MODE=chunked timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2 > $T/tests_chunked.txt
