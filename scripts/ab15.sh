#!/bin/bash
# Bisect the last-CTA tails (TTG_LZ_TAILS bitmask) and the L2 prefetch distance on config 3.
O=gpurun_out/ab15
mkdir -p $O
for T in 0 1 2 4 7; do
  TTG_LZ_PD=0 TTG_LZ_TAILS=$T timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "config3" > $O/pytest_tails$T.txt 2>&1
  echo "exit $?" >> $O/pytest_tails$T.txt
done
for PD in 0 2 4 8; do
  TTG_LZ_PD=$PD TTG_LZ_TAILS=0 timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/bench_pd$PD.json 2> $O/bench_pd$PD.err
done
echo done
