#!/bin/bash
# Round profile pass (GPU box): bench lines for every BASELINE config, the config-4 loop,
# the ncu launch list of the default bench and a full ncu capture of the dominant kernel.
O=gpurun_out/r1b
mkdir -p $O
timeout 300 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
for c in 1 3 5; do timeout 400 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
timeout 300 python scripts/try_cfg4_loop.py 20 > $O/cfg4_loop_20iters.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_cfg2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass1_big -c 4 -o $O/big_cfg2 \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
