#!/bin/bash
# A/B of the HostEnergySweep ordering inside bench.py (same box): default vs the
# previous behaviour (first energy streamed, last energy drained whole).
for v in "" "BSEL_SWEEP_STREAM_FIRST=1 BSEL_SWEEP_STREAM_LAST=0" "" "BSEL_SWEEP_STREAM_FIRST=1 BSEL_SWEEP_STREAM_LAST=0"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-cfg5 --no-other-b --no-seq 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'single', round(d['e2e']['single_call_ms'],1))"
done
