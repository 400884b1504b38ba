#!/bin/bash
# Candidate engine with the explicit-Q reflector for 512 <= k <= 2048: parity, config 5 / 3 benches.
O=gpurun_out/ab22
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py tests/test_gpu_engines.py tests/test_gpu_sweeps.py -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?" >> $O/pytest.txt
timeout 600 python bench.py --config 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
TTG_PHASES=1 timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 2 --warmup 1 --e2e-concurrency 1 > $O/bench_cfg5_phases.json 2> $O/bench_cfg5_phases.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_cfg5_launches.csv \
  python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu5.log 2>&1
echo done
