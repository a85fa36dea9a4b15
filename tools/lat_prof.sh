#!/bin/bash
# Single-image latency: per-kernel device times of configs 1 and 3 (launch list) beside the
# bench's per-step time.  Usage: tools/lat_prof.sh <tag>
TAG=${1:-lat}
mkdir -p gpurun_out
for CFG in cfg1 cfg3; do
  python bench.py --config $CFG --e2e-steps 0 --no-cpu-baseline > gpurun_out/lat_b_${TAG}_$CFG.log 2>&1
  tail -1 gpurun_out/lat_b_${TAG}_$CFG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', d['ms_per_step'], d['roofline']['pipeline']['phase_ms'])"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/lat_l_${TAG}_$CFG.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > /dev/null 2>&1
done
