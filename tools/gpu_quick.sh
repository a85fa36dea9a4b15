#!/bin/bash
# Quick GPU check of a build: the parity-heavy GPU tests, then the cfg2 bench without the
# e2e/CPU legs (phase times).  Usage: tools/gpu_quick.sh <tag> [pytest -k expr]
TAG=${1:-q}; K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?"
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?"
fi
tail -3 gpurun_out/t_$TAG.log
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_$TAG.log 2>&1; echo "bench rc=$?"
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
lines = open(f"gpurun_out/b_{tag}.log").read().strip().splitlines()
try:
    d = json.loads(lines[-1])
    print("value", round(d["value"], 2), "ms", round(d["ms_per_step"], 4), d["roofline"]["pipeline"]["phase_ms"], d["parity"]["summary"])
except Exception as e:
    print("\n".join(lines[-20:]))
PY
