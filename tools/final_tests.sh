#!/bin/bash
# Final verification on a 4-GPU box: the whole GPU suite (incl. the world-4
# NCCL tests), smoke, and the reference arm of bench.py.
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests_final4.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err
tail -1 gpurun_out/smoke_final.log; tail -3 gpurun_out/gputests_final4.log; tail -c 600 gpurun_out/ref_arm.json
