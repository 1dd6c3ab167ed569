#!/bin/bash
# One profiling call on the GPU box: PCIe roofline, bench launch list, ncu --set full captures of
# the hot kernels (513^3 fp32, the bench workload, device-resident as in the kernel-only leg).
# Outputs under gpurun_out/prof/.
O=gpurun_out/prof
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
python tools/pcie_bw.py 1024 > $O/pcie.json 2>&1
# launches of the bench command with their device time (cold-cache, serialised); the first 1500
# cover the kernel-only compress/decompress legs and the M1 legs
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --zfp-rate 0 > $O/bench_under_ncu.log 2>&1
D="python tools/prof_driver_dev.py 513"
N="timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$N -k "regex:k_level_pass1<\(int\)2, \(bool\)1, \(bool\)1, \(bool\)1, float>" -s 1 -c 1 -o $O/pass1q $D > /dev/null 2>&1
$N -k "regex:k_decode_warp" -s 1 -c 1 -o $O/decode $D > /dev/null 2>&1
$N -k "regex:k_level_final<\(bool\)1, \(bool\)1, \(bool\)1, float>" -s 1 -c 1 -o $O/final $D > /dev/null 2>&1
$N -k "regex:k_level_pass2" -s 9 -c 1 -o $O/pass2 $D > /dev/null 2>&1
$N -k "regex:k_level_pass1_2r<\(int\)1" -s 1 -c 1 -o $O/pass1r $D > /dev/null 2>&1
$N -k "regex:k_thomas" -s 0 -c 3 -o $O/thomas $D > /dev/null 2>&1
$N -k "regex:k_encode" -s 1 -c 1 -o $O/encode $D > /dev/null 2>&1
$N -k "regex:k_minmax" -s 1 -c 1 -o $O/minmax $D > /dev/null 2>&1
ls -la $O
