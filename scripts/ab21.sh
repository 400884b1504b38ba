#!/bin/bash
# Final candidate-engine settings (pd by width, cap by width, resid by width): all GPU tests, benches.
O=gpurun_out/ab21
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
TTG_PHASES=1 timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 2 --warmup 1 --e2e-concurrency 1 > $O/bench_cfg5_phases.json 2> $O/bench_cfg5_phases.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg5_launches.csv \
  python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu5.log 2>&1
echo done
