#!/bin/bash
# tails = 5 (threshold + next first choice as last-CTA tails), L2 prefetch distance 2, pipelined e2e:
# all GPU tests, bench lines.
O=gpurun_out/ab16
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_LZ_TAILS=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_tails0.json 2> $O/bench_cfg3_tails0.err
timeout 600 python bench.py --config 5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 --e2e-concurrency 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu3.log 2>&1
echo done
