#!/bin/bash
# Candidate engine up to k = 1024 (config 5's first cut): parity and A/B against the subspace engine.
O=gpurun_out/ab19
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py tests/test_gpu_engines.py -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?" >> $O/pytest.txt
timeout 600 python bench.py --config 5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
TTG_LAZY_WIDE=0 timeout 600 python bench.py --config 5 --no-cpu-baseline > $O/bench_cfg5_sub.json 2> $O/bench_cfg5_sub.err
TTG_LZW_CAP=4096 timeout 600 python bench.py --config 5 --no-cpu-baseline > $O/bench_cfg5_cap4k.json 2> $O/bench_cfg5_cap4k.err
TTG_PHASES=1 timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 2 --warmup 1 --e2e-concurrency 1 > $O/bench_cfg5_phases.json 2> $O/bench_cfg5_phases.err
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
echo done
