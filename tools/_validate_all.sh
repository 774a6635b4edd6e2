mkdir -p gpurun_out/val
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/val/gpu_tests.log 2>&1; tail -1 gpurun_out/val/gpu_tests.log
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 5 2>&1 | tail -1 > gpurun_out/val/bench_c$c.json; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/val/ref.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/val/torchrun.json
for f in gpurun_out/val/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d.get('impl','ours'), d.get('value'), d.get('unit'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), d.get('latency_ms'))"; done
