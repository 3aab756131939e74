#!/bin/bash
# Inverse phase statistics alone (instrumented build) for build variants: tools/coloc_probe.sh "-DX=1" ...
for v in "" "$@"; do
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 EXTRA="-DBSEL_INV_STATS=1 $v" >/dev/null 2>&1
for df in 1 0; do for g in 64 2; do BSEL_INV_DATAFLOW=$df BSEL_INV_GRID=$g BSEL_INV_STATS=1 timeout 300 python tools/inv_probe.py 2>&1 | grep "inverse stats" | grep -v "SMs used" | sed "s/^/[$v] df $df grid $g: /"; done; done
done
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
