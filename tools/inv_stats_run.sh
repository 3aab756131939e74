#!/bin/bash
# Per-phase statistics of the persistent inverse (instrumented build,
# -DBSEL_INV_STATS=1): alone (tools/inv_probe.py), in the 1-GPU cfg4 step and
# in the 2-GPU step, for the dataflow (default) and the barrier kernel.
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 EXTRA=-DBSEL_INV_STATS=1 >/dev/null 2>&1
for df in 1 0; do
  echo "== BSEL_INV_DATAFLOW=$df"
  BSEL_INV_DATAFLOW=$df BSEL_INV_STATS=1 timeout 300 python tools/inv_probe.py 2>&1 | grep "inverse stats" | sed 's/^/alone: /'
  BSEL_INV_DATAFLOW=$df BSEL_INV_STATS=1 timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-other-b --no-seq --no-cfg5 2>&1 >/dev/null | grep "inverse stats" | sed 's/^/1gpu: /'
  if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
    BSEL_INV_DATAFLOW=$df BSEL_INV_STATS=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29630 + df)) bench.py --gpus 2 --steps 3 --warmup 2 --no-e2e 2>&1 >/dev/null | grep "inverse stats" | sed 's/^/2gpu: /'
  fi
done
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
