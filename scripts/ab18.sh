#!/bin/bash
# Exact pass with the fragment-layout epilogue (no staging), tails = 7, per-step-join e2e: parity, bench x3, ncu.
O=gpurun_out/ab18
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py tests/test_gpu_engines.py -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?" >> $O/pytest.txt
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_r$i.json 2> $O/bench_cfg3_r$i.err
done
TTG_LZ_PD=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_pd0.json 2> $O/bench_cfg3_pd0.err
TTG_LZ_PD=3 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_pd3.json 2> $O/bench_cfg3_pd3.err
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_lzw_refresh_mma" --launch-skip 12 --launch-count 1 \
  -o $O/ncu_full_narrow python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu_full.log 2>&1
echo done
