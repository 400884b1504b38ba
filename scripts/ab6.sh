#!/bin/bash
# Candidate pivoting timings (config 3) + engine alternatives; config-4 default routing.
O=gpurun_out/ab7
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_engines.py -q -p no:cacheprovider > $O/pytest_lazy_engines.txt 2>&1
echo "exit $?" >> $O/pytest_lazy_engines.txt
timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err

timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu3.log 2>&1
echo done
