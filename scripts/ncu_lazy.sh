#!/bin/bash
# Candidate pivoting: parity, bench, and ncu --set full of an exact pass and the per-step kernels.
O=gpurun_out/ncu_lazy2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lazy.py -q -p no:cacheprovider > $O/pytest_lazy.txt 2>&1
echo "exit $?" >> $O/pytest_lazy.txt
timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TTG_PHASES=1 timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 > $O/bench_cfg3_phases.json 2> $O/bench_cfg3_phases.err
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_lz_refresh" --launch-skip 12 --launch-count 1 \
  -o $O/refresh python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_refresh.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_lz_gather|k_lz_update|k_wy_fused_smem|k_sub_prep" --launch-skip 6 --launch-count 8 \
  -o $O/small python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_small.log 2>&1
echo done
