#!/bin/bash
# Merged lazy-step tails (threshold, final choice, next first choice as last-CTA tails), upload /
# device turn locks, gram unroll: all GPU tests, bench, member-cap experiments.
O=gpurun_out/ab14
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_LZ_CAP=262144 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_cap262k.json 2> $O/bench_cfg3_cap262k.err
TTG_LZ_CAP=16384 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_cap16k.json 2> $O/bench_cfg3_cap16k.err
TTG_LZW_CAP=4096 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_wcap4k.json 2> $O/bench_cfg3_wcap4k.err
TTG_LZW_CAP=65536 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_wcap64k.json 2> $O/bench_cfg3_wcap64k.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 --e2e-concurrency 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu3.log 2>&1
echo done
