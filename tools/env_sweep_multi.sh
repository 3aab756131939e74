#!/bin/bash
# tools/env_sweep_multi.sh N "ENV=..." ... : cfg4 step on N GPUs per variant (torchrun).
N=$1; shift
port=29600
for v in "" "$@"; do
  port=$((port + 1))
  out=$(env $v timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $N --steps 3 --warmup 2 --no-e2e 2>/dev/null)
  echo "$out" | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value'],1), {k: round(x,1) for k,x in d['phases_ms'].items()})
except Exception as e: print('${v:-default}', 'failed', e)"
done
