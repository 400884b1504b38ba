#!/bin/bash
# cp.async exact pass + concurrent device timing in bench (config 3).
O=gpurun_out/ab9
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py -k "lazy or config3" -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?" >> $O/pytest.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_lz_refresh" --launch-skip 12 --launch-count 1 \
  -o $O/ncu_full_lz_refresh python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu_full.log 2>&1
echo done
