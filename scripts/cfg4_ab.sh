#!/bin/bash
# Config-4 A/B: blocked in-place engine vs per-step launches (TTG_TALL_UNBLOCKED=1); parity
# tests on the in-place engine; phase totals and the ncu launch list of one decomposition.
O=gpurun_out/cfg4ab
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sweeps.py -k "qr_col_pivot" -x -q -p no:cacheprovider > $O/pytest_qrcp.txt 2>&1
echo "exit $?" >> $O/pytest_qrcp.txt
TTG_CUT_TIMING=1 timeout 300 python scripts/try_cfg4.py 2 > $O/cut_timing_blocked.txt 2>&1
TTG_PHASES=1 timeout 300 python scripts/try_cfg4.py 1 > $O/phases_blocked.txt 2>&1
TTG_TALL_UNBLOCKED=1 TTG_CUT_TIMING=1 timeout 300 python scripts/try_cfg4.py 2 > $O/cut_timing_steps.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_completion.py tests/test_gpu_fullsize.py -k "config4 or half_observed or rank_adaptive" -x -q -p no:cacheprovider > $O/pytest_cfg4.txt 2>&1
echo "exit $?" >> $O/pytest_cfg4.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg4_launches.csv \
  python scripts/try_cfg4.py 1 > $O/ncu.log 2>&1
echo done
