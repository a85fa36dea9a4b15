#!/bin/bash
# One GPU call: plain bench (must exit 0 first), then the launch list and one --set full capture
# of the tile kernels.  Usage: tools/capture_round.sh <tag> [config]
set -u
TAG=$1; CFG=${2:-cfg2}
mkdir -p gpurun_out
python bench.py --config $CFG > gpurun_out/bench_$TAG.log 2>&1 || { echo "bench failed"; tail -20 gpurun_out/bench_$TAG.log; exit 1; }
tail -1 gpurun_out/bench_$TAG.log
# the kernel profiles cover the whole batch as one pipeline (the roofline's phase times do too)
export RUNLAB_GPU_SPLIT=1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --config $CFG --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity \
    > gpurun_out/ncu_l_$TAG.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_analyze|k_emit" -c 6 -o gpurun_out/prof_$TAG -f \
    python bench.py --config $CFG --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture rc=$?"
