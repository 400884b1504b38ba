#!/bin/bash
# tails = 7 with the wide-guard fix, chunked upload, hist/gather two strips per trip: parity, e2e stability.
O=gpurun_out/ab17
mkdir -p $O
TTG_LZ_TAILS=7 timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "lazy or config3" > $O/pytest_tails7.txt 2>&1
echo "exit $?" >> $O/pytest_tails7.txt
timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py tests/test_gpu_engines.py -q -p no:cacheprovider > $O/pytest_default.txt 2>&1
echo "exit $?" >> $O/pytest_default.txt
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_r$i.json 2> $O/bench_cfg3_r$i.err
done
for i in 1 2; do
  TTG_LZ_TAILS=7 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_tails7_r$i.json 2> $O/bench_cfg3_tails7_r$i.err
done
echo done
