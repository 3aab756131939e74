#!/bin/bash
# tools/build_sweep_multi.sh N "-DX=1" ... : rebuild with compile-time knobs, cfg4 step on N GPUs (torchrun).
N=$1; shift
port=29800
for v in "" "$@"; do
  make -C paper_2601_04904_b200/csrc clean >/dev/null
  make -C paper_2601_04904_b200/csrc -j16 EXTRA="$v" >/dev/null 2>&1 || { echo "$v build failed"; continue; }
  port=$((port + 1))
  out=$(timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $N --steps 3 --warmup 2 --no-e2e 2>/dev/null)
  echo "$out" | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value'],1), {k: round(x,1) for k,x in d['phases_ms'].items()})
except Exception as e: print('${v:-default}', 'failed', e)"
done
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
