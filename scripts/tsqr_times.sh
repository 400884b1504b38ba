# usage: bash scripts/tsqr_times.sh  (on the GPU box) -> TSQR/small_qrcp launch times of one cfg2 ULV decomposition
python scripts/one_decomp.py 2 ulv 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg2_ulv_launches.csv -k regex:tsqr python scripts/one_decomp.py 2 ulv 1 > gpurun_out/ncu.log 2>&1
