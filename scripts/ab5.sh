#!/bin/bash
# In-place engines on config 4: persistent blocked (default) vs per-step kernels.
O=gpurun_out/ab5
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sweeps.py -k "qr_col_pivot" -x -q -p no:cacheprovider > $O/pytest_qrcp.txt 2>&1
echo "exit $?" >> $O/pytest_qrcp.txt
TTG_CUT_TIMING=1 timeout 300 python scripts/try_cfg4.py 2 > $O/cfg4_cut_timing.txt 2>&1
TTG_TALL_ENGINE=steps TTG_CUT_TIMING=1 timeout 300 python scripts/try_cfg4.py 2 > $O/cfg4_cut_timing_steps.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_completion.py tests/test_gpu_fullsize.py -k "config4 or half_observed or rank_adaptive" -x -q -p no:cacheprovider > $O/pytest_cfg4.txt 2>&1
echo "exit $?" >> $O/pytest_cfg4.txt
timeout 400 python scripts/cfg4_loop.py 20 > $O/cfg4_loop_20iters.txt 2>&1

timeout 900 python -m pytest tests/test_gpu_lazy.py -q -p no:cacheprovider > $O/pytest_lazy.txt 2>&1
echo "exit $?" >> $O/pytest_lazy.txt
timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err
echo done
