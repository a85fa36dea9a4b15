#!/bin/bash
# A/B of env knobs on the device bench: tools/ab_env.sh "cfg1 cfg3 cfg2" "base;RUNLAB_GPU_NO_PDL=1" [reps]
CFGS=$1; VARS=$2; REPS=${3:-2}
mkdir -p gpurun_out
IFS=';' read -ra VA <<< "$VARS"
for r in $(seq $REPS); do
for CFG in $CFGS; do
  for V in "${VA[@]}"; do
    if [ "$V" = base ]; then E=""; else E="$V"; fi
    env $E python bench.py --config $CFG --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$CFG', '$V', round(d['ms_per_step'],4), round(d['value'],2), {k: round(v,4) for k,v in d['roofline']['pipeline']['phase_ms'].items()})
except Exception as e: print('$CFG $V FAILED', e)"
  done
done
done
