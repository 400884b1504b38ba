#!/bin/bash
# Same-box A/B of three builds on config 3 (old: division-based prefetch bookkeeping; new: incremental;
# cur: + 512-thread pass for k > 512) and config 5 member caps with the current build.
O=gpurun_out/ab20
mkdir -p $O
L=paper_2501_07904_b200/lib
for v in old new cur old new cur; do
  cp $L/ab_$v.so $L/libttutv_b200.so
  timeout 600 python bench.py --no-cpu-baseline --steps 6 > $O/bench_cfg3_${v}_$RANDOM.json 2>> $O/bench_cfg3.err
done
cp $L/ab_cur.so $L/libttutv_b200.so
timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?" >> $O/pytest.txt
timeout 600 python bench.py --config 5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for C in 2048 4096 16384; do
  TTG_LZW_CAP=$C timeout 600 python bench.py --config 5 --no-cpu-baseline --steps 5 > $O/bench_cfg5_cap$C.json 2> $O/bench_cfg5_cap$C.err
done
TTG_LZ_PD=0 timeout 600 python bench.py --config 5 --no-cpu-baseline --steps 5 > $O/bench_cfg5_pd0.json 2> $O/bench_cfg5_pd0.err
TTG_LZ_PD=4 timeout 600 python bench.py --config 5 --no-cpu-baseline --steps 5 > $O/bench_cfg5_pd4.json 2> $O/bench_cfg5_pd4.err
echo done
