#!/bin/bash
# Inverse: event-timed span per launch (BSEL_PROFILE_DUMP timeline of the profiled
# step) vs the kernel's own duration (instrumented build, BSEL_INV_STATS), cfg4 1 GPU.
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 EXTRA=-DBSEL_INV_STATS=1 >/dev/null 2>&1
BSEL_INV_STATS=1 BSEL_PROFILE_DUMP=gpurun_out/tl_gap.csv timeout 400 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-other-b --no-seq --no-cfg5 2>&1 >/dev/null | grep "inverse stats" | grep -v SMs
python tools/timeline_stats.py gpurun_out/tl_gap.csv
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
