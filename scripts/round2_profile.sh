#!/bin/bash
# Round-2 profile pass (GPU box): all GPU tests, smoke, bench lines for configs 3 (headline),
# 5, 2, 1, the reference arm, the config-4 loop, the ncu launch list of the headline bench and
# ncu --set full captures of its dominant kernel (a non-idle exact pass of the candidate engine, on DMMA)
# and of the pipelined DMMA GEMM.
O=gpurun_out/r2d
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 python bench.py --config 2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --config 1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 400 python scripts/cfg4_loop.py 20 > $O/cfg4_loop_20iters.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_cfg3_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_lzw_refresh_mma" --launch-skip 12 --launch-count 1 \
  -o $O/ncu_full_lzw_refresh_mma python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-concurrency 1 > $O/ncu_full.log 2>&1
timeout 600 python scripts/gemm_throughput.py > $O/gemm.json 2> $O/gemm.err
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_gemm128" --launch-skip 2 --launch-count 1 \
  -o $O/ncu_full_gemm128 python scripts/gemm_throughput.py > $O/ncu_gemm.log 2>&1
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_cfg3.json 2> $O/bench_ref_cfg3.err
echo done
