#!/bin/bash
# Wide candidate exact pass on DMMA: parity (lazy tests, full-size config 3), bench, launch list.
O=gpurun_out/ab12
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "lazy or config3" > $O/pytest.txt 2>&1
echo "exit $?" >> $O/pytest.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 --e2e-concurrency 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu3.log 2>&1
echo done
