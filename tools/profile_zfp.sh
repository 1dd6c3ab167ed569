#!/bin/bash
# Fixed-rate coder captures (513^3 fp32, rate 16 -- the bench's zfp leg) plus the bench launch list.
O=gpurun_out/profz
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
N="timeout 600 ncu --set full --clock-control none --import-source on"
$N -k regex:k_zfp_encode -s 3 -c 1 -o $O/k_zfp_encode python tools/zfp_kbench.py 16 > /dev/null 2>&1
$N -k regex:k_zfp_decode -s 3 -c 1 -o $O/k_zfp_decode python tools/zfp_kbench.py 16 > /dev/null 2>&1
ls -la $O
