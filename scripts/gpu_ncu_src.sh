#!/bin/bash
# usage: gpu_ncu_src.sh cfg kernel_regex tag   -> gpurun_out/src_<tag>.csv (+ .ncu-rep)
mkdir -p gpurun_out
cfg=$1; k=$2; tag=$3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -f -o gpurun_out/src_$tag \
  python scripts/profile_run.py $cfg 6 > gpurun_out/src_$tag.log 2>&1
ncu -i gpurun_out/src_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$tag.csv 2>>gpurun_out/src_$tag.log
