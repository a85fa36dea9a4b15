#!/bin/bash
# Source-level ncu of one kernel launch (after the warm-up call): tools/src_prof2.sh <tag> <cells> <kernel> [skip]
TAG=$1; CELLS=$2; K=$3; SKIP=${4:-1}
mkdir -p gpurun_out
export RUNLAB_GPU_SPLIT=1
ncu --set full --import-source on --clock-control none -k "$K" --launch-skip $SKIP -c 1 -o gpurun_out/src_$TAG -f \
  python tools/prof_driver.py --cells $CELLS --copies 8 --iters 2 > gpurun_out/sp_ncu_$TAG.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/src_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_${TAG}.csv 2>/dev/null
ncu -i gpurun_out/src_$TAG.ncu-rep --page details --csv > gpurun_out/src_${TAG}_details.csv 2>/dev/null
