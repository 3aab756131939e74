#!/bin/bash
# torchrun --no-python target: each rank dumps its profiled step's per-launch
# timeline to gpurun_out/tl_rank$LOCAL_RANK.csv (analysed by tools/timeline_stats.py).
exec env BSEL_PROFILE_DUMP=gpurun_out/tl_rank${LOCAL_RANK}.csv python bench.py "$@"
