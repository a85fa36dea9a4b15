#!/bin/bash
# A/B of library builds on the device bench (3 pipelines): tools/ab_bench.sh "cur new" "cfg2 cfg1" [reps]
LIBS=$1; CFGS=${2:-cfg2}; REPS=${3:-2}
for r in $(seq $REPS); do for C in $CFGS; do for L in $LIBS; do
RUNLAB_GPU_LIB=$PWD/paper_2006_09299_b200/librunlab_gpu_$L.so python bench.py --config $C --e2e-steps 0 --no-cpu-baseline --no-parity > /tmp/b.log 2>&1
tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', '$L', round(d['ms_per_step'],4), round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['pipeline']['phase_ms'].items()})" || tail -3 /tmp/b.log
done; done; done
