#!/bin/bash
# Source-level ncu profile of chosen kernels on a device-generated batch of chosen cells.
# Usage: tools/src_prof.sh <tag> <cells d:g,...> <kernel regex> [count]
TAG=$1; CELLS=$2; KRE=$3; CNT=${4:-2}
mkdir -p gpurun_out
export RUNLAB_GPU_SPLIT=1
python tools/prof_driver.py --cells $CELLS --copies 8 --iters 3 > gpurun_out/sp_time_$TAG.log 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k regex:"$KRE" -c $CNT -o gpurun_out/src_$TAG -f \
  python tools/prof_driver.py --cells $CELLS --copies 8 --iters 1 > gpurun_out/sp_ncu_$TAG.log 2>&1; echo ncu rc=$?
for k in $(echo "$KRE" | tr '|' ' ' | tr -d '$^'); do
  ncu -i gpurun_out/src_$TAG.ncu-rep -k $k --page source --csv --print-source cuda,sass > gpurun_out/src_${TAG}_$k.csv 2>/dev/null
done
ncu -i gpurun_out/src_$TAG.ncu-rep --page details --csv > gpurun_out/src_${TAG}_details.csv 2>/dev/null
