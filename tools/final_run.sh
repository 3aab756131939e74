set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests_final.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/g1.json 2> gpurun_out/g1.err
timeout 800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/g4.json 2> gpurun_out/g4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/g2.json 2> gpurun_out/g2.err
tail -2 gpurun_out/smoke_final.log; tail -3 gpurun_out/gputests_final.log
python -c "
import json
for f in ('gpurun_out/g1.json','gpurun_out/g2.json','gpurun_out/g4.json'):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['value'],1), {k: round(v,1) for k,v in d['phases_ms'].items()}, 'e2e', d.get('e2e',{}).get('value'), d.get('clocks',{}).get('reasons'), (d.get('config5') or {}).get('ms_per_energy'), d.get('partition_sizes'))
    except Exception as e: print(f, 'fail', e)
"
