#!/bin/bash
# tools/src_sweep_multi.sh N dir1 dir2 ... : per variant, overlay the source files of
# dirK onto csrc/, rebuild, time the cfg4 step on N GPUs (torchrun); csrc restored after.
N=$1; shift
C=paper_2601_04904_b200/csrc
mkdir -p /tmp/csrc_orig && cp $C/*.cu $C/*.cuh /tmp/csrc_orig/
port=29700
for v in "" "$@"; do
  cp /tmp/csrc_orig/* $C/
  [ -n "$v" ] && cp $v/* $C/
  make -C $C clean >/dev/null; make -C $C -j16 >/dev/null 2>&1 || { echo "$v build failed"; continue; }
  for rep in 1 2; do
    port=$((port + 1))
    out=$(timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
          --master-port $port bench.py --gpus $N --steps 3 --warmup 2 --no-e2e 2>/dev/null)
    echo "$out" | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value'],1), {k: round(x,1) for k,x in d['phases_ms'].items()})
except Exception as e: print('${v:-default}', 'failed', e)"
  done
done
cp /tmp/csrc_orig/* $C/
make -C $C clean >/dev/null; make -C $C -j16 >/dev/null 2>&1
