#!/bin/bash
# Final check of the head: all GPU tests, smoke, headline bench line (with the CPU baseline), config 5.
O=gpurun_out/ab25
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_cfg3_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo done
