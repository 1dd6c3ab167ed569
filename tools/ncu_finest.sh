#!/bin/bash
# ncu --set full captures of the finest-level launch of each hot kernel (513^3 fp32 driver:
# compress, decompress, compress, decompress -> the second pass is captured).
set -x
OUT=${1:-gpurun_out/prof}
D="python tools/prof_driver.py 513"
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:k_level_pass1sILi2ELb1ELb1ELb1EfE -s 1 -c 1 -o ${OUT}_pass1q $D
$N -k regex:k_level_pass2 -s 18 -c 1 -o ${OUT}_pass2 $D
$N -k regex:k_decode -s 1 -c 1 -o ${OUT}_decode $D
$N -k regex:k_level_finalILb1ELb1ELb1EfE -s 1 -c 1 -o ${OUT}_final $D
$N -k regex:k_level_pass1ILi1ELb1ELb1ELb1EdE -s 17 -c 1 -o ${OUT}_pass1r $D
$N -k regex:k_thomas_reg -s 54 -c 3 -o ${OUT}_thomas $D
