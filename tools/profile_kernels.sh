#!/bin/bash
# ncu --set full captures of the finest-level launch of each hot kernel (bench workload, 513^3).
O=${1:-gpurun_out/prof2}
mkdir -p $O
export HPDR_NO_STREAM_DECODE=1
D="python tools/prof_driver_dev.py 513"
N="timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:k_level_pass1ILi2ELb1ELb1ELb1EfE -s 2 -c 1 -o $O/pass1q $D > /dev/null 2>&1
$N -k regex:k_level_pass1ILi1E -s 9 -c 1 -o $O/pass1r $D > /dev/null 2>&1
$N -k regex:k_level_pass2 -s 27 -c 1 -o $O/pass2 $D > /dev/null 2>&1
$N -k regex:k_level_final -s 17 -c 1 -o $O/final $D > $O/final.log 2>&1
$N -k regex:k_decode_warp -s 1 -c 1 -o $O/decode $D > $O/decode.log 2>&1
$N -k regex:k_thomas -s 81 -c 3 -o $O/thomas $D > /dev/null 2>&1
$N -k regex:k_encode -s 2 -c 1 -o $O/encode $D > $O/encode.log 2>&1
ls $O
