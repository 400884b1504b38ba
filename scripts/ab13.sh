#!/bin/bash
# Narrow candidate exact pass on DMMA (A/B against the cp.async FMA pass), wide member update v2.
O=gpurun_out/ab13
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "lazy or config3" > $O/pytest.txt 2>&1
echo "exit $?" >> $O/pytest.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_LZ_MMA=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_fma.json 2> $O/bench_cfg3_fma.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 --e2e-concurrency 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_lzw_refresh_mma" --launch-skip 12 --launch-count 1 \
  -o $O/ncu_full_narrow python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu_full.log 2>&1
echo done
