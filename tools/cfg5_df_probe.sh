./tools/inv_micro | grep -E '"n": (512|1024)'
BSEL_INV_DATAFLOW=0 ./tools/inv_micro | grep -E '"n": (512|1024)'
for df in 1 0; do
  BSEL_INV_DATAFLOW=$df timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-other-b --no-seq 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('df $df', d['value'], d['config5']['ms_per_energy'])"
done
