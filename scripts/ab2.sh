#!/bin/bash
# Candidate pivoting (config 3) checks + timings; blocked vs per-step in-place engine (config 4).
O=gpurun_out/ab4
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lazy.py -q -p no:cacheprovider > $O/pytest_lazy.txt 2>&1
echo "exit $?" >> $O/pytest_lazy.txt
timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -k "config3" -x -q -p no:cacheprovider > $O/pytest_full3.txt 2>&1
echo "exit $?" >> $O/pytest_full3.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu3.log 2>&1
echo done
