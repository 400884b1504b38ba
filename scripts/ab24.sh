#!/bin/bash
# Member-cap sweep on config 3 (narrow and wide caps), same box.
O=gpurun_out/ab24
mkdir -p $O
for C in 65536 16384 32768 131072 65536; do
  TTG_LZ_CAP=$C timeout 600 python bench.py --no-cpu-baseline --steps 6 --e2e-concurrency 1 > $O/bench_cap${C}_$RANDOM.json 2>> $O/err.txt
done
for C in 16384 4096 8192 16384; do
  TTG_LZW_CAP=$C timeout 600 python bench.py --no-cpu-baseline --steps 6 --e2e-concurrency 1 > $O/bench_wcap${C}_$RANDOM.json 2>> $O/err.txt
done
echo done
