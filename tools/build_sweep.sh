#!/bin/bash
# Rebuild the library with compile-time knobs and time the cfg4 1-GPU step per variant (GPU box):
#   tools/build_sweep.sh "-DBSEL_BARRIER_SLEEP=0" "-DBSEL_TILE_ACC=1" ...
for v in "" "$@"; do
  make -C paper_2601_04904_b200/csrc clean >/dev/null
  make -C paper_2601_04904_b200/csrc -j16 EXTRA="$v" >/dev/null 2>&1 || { echo "$v build failed"; continue; }
  out=$(timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-other-b --no-seq 2>/dev/null)
  echo "$out" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value'],1), {k: round(x,1) for k,x in d['phases_ms'].items()})"
done
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
