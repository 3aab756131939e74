timeout 300 python -m pytest tests/test_gpu_seq.py -x -q -k "inverse" 2>&1 | tail -3
BSEL_INV_DATAFLOW=0 timeout 120 ./tools/inv_micro 2>&1 | grep inverse_us
timeout 120 ./tools/inv_micro 2>&1 | grep -E "inverse_us|err"
tools/env_sweep.sh BSEL_INV_DATAFLOW=0
tools/env_sweep_multi.sh 2 BSEL_INV_DATAFLOW=0
