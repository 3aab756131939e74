#!/bin/bash
# Rebuild the library with compile-time knobs; per variant: the isolated
# inverse (tools/inv_micro, n = 512 / 1024) and the cfg4 1-GPU step (GPU box):
#   tools/build_sweep.sh "-DBSEL_BARRIER_SLEEP=0" "-DBSEL_TILE_ACC=1" ...
O=paper_2601_04904_b200/csrc/build
for v in "" "$@"; do
  make -C paper_2601_04904_b200/csrc clean >/dev/null
  make -C paper_2601_04904_b200/csrc -j16 EXTRA="$v" >/dev/null 2>&1 || { echo "$v build failed"; continue; }
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/inv_micro_v tools/inv_micro.cu \
    $O/inverse.o $O/zgemm.o $O/zgemm3m.o $O/publish.o -lcuda >/dev/null 2>&1 &&
    timeout 120 /tmp/inv_micro_v 2>/dev/null | grep -E '"n": (512|1024)' | tr '\n' ' ' | sed "s/^/${v:-default} inverse: /"; echo
  [ -n "$NO_STEP" ] && continue
  out=$(timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-other-b --no-seq --no-cfg5 2>/dev/null)
  echo "$out" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value'],1), {k: round(x,1) for k,x in d['phases_ms'].items()})"
done
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
