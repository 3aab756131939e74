#!/bin/bash
# Chain launch gaps and inverse phases at 2 GPUs (instrumented build), PDL on / off.
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 EXTRA=-DBSEL_INV_STATS=1 >/dev/null 2>&1
for pdl in 1 0; do
  BSEL_INV_PDL=$pdl BSEL_INV_STATS=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29650 + pdl)) bench.py --gpus 2 --steps 3 --warmup 2 --no-e2e 2>&1 >/dev/null | grep "inverse stats" | grep -v SMs | sed "s/^/pdl $pdl: /"
done
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
