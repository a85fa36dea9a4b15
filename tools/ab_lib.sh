#!/bin/bash
# A/B of library builds on chosen cells (one pipeline, phase times): tools/ab_lib.sh "base new" "0.5:1 0.5:4 cfg2" [reps]
LIBS=$1; CELLS=$2; REPS=${3:-3}
export RUNLAB_GPU_SPLIT=1
for r in $(seq $REPS); do
for C in $CELLS; do
  for L in $LIBS; do
    if [ "$C" = cfg2 ]; then A="--cfg2"; else A="--cells $C --copies 16"; fi
    RUNLAB_GPU_LIB=$PWD/paper_2006_09299_b200/librunlab_gpu_$L.so python tools/prof_driver.py $A --iters 5 > /tmp/ab_one.log 2>&1
    tail -1 /tmp/ab_one.log | python -c "import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$C', '$L', *(f\"{k[:-3]} {d[k]:.4f}\" for k in ('analyze_ms','merge_ms','emit_ms','total_ms')))
except Exception as e: print('$C $L FAILED', e)" || true
    grep -q '"images"' /tmp/ab_one.log || tail -5 /tmp/ab_one.log
  done
done
done
