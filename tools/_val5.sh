mkdir -p gpurun_out/val5
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/val5/bench_c2.json 2> gpurun_out/val5/bench_c2.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/val5/ref.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/val5/torchrun.json 2>&1
for f in gpurun_out/val5/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('impl','ours'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), d.get('gpu_launches'))"; done
