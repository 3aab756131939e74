#!/bin/bash
# Time the cfg4 1-GPU step under environment-knob variants (GPU box):
#   tools/env_sweep.sh "BSEL_SCHUR=1" "BSEL_LANE_INV_GRID=48" ...
# One line per variant: value (ms) and forward / backward phases.
for v in "" "$@"; do
  out=$(env $v timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-other-b --no-seq --no-cfg5 2>/dev/null)
  echo "$out" | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value'],1), {k: round(x,1) for k,x in d['phases_ms'].items()})
except Exception as e: print('${v:-default}', 'failed', e)"
done
