#!/bin/bash
# One profiling call on the GPU box: PCIe roofline, bench launch list, ncu --set full captures of
# the hot kernels (513^3 fp32, the bench workload).  Outputs under gpurun_out/prof/.
O=gpurun_out/prof
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
python tools/pcie_bw.py 1024 > $O/pcie.json 2>&1
# every launch of the bench command with its device time (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
D="python tools/prof_driver.py 513"
N="timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:k_level_pass1ILi2ELb1ELb1ELb1EfE -s 1 -c 1 -o $O/pass1q $D > /dev/null 2>&1
$N -k regex:k_decode -s 1 -c 1 -o $O/decode $D > /dev/null 2>&1
$N -k regex:k_level_finalILb1ELb1ELb1EfE -s 1 -c 1 -o $O/final $D > /dev/null 2>&1
$N -k regex:k_level_pass2 -s 18 -c 1 -o $O/pass2 $D > /dev/null 2>&1
$N -k regex:k_level_pass1ILi1ELb1ELb1ELb1EdE -s 17 -c 1 -o $O/pass1r $D > /dev/null 2>&1
$N -k regex:k_thomas -s 54 -c 3 -o $O/thomas $D > /dev/null 2>&1
$N -k regex:k_encode -s 1 -c 1 -o $O/encode $D > /dev/null 2>&1
ls -la $O
