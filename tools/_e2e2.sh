timeout 600 python -m pytest tests -q -m gpu -x -k "host or cpu_tensors or export or reload" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-steps 0 --unshuffle-steps 0 --fp32-fast-steps 0 > gpurun_out/e2e2.json 2>gpurun_out/e2e2.err; python -c "
import json; d=json.loads(open('gpurun_out/e2e2.json').read().strip().splitlines()[-1]); print('bench', d['value'], 'e2e', d['e2e'])"
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --fp32-steps 0 --unshuffle-steps 0 --fp32-fast-steps 0 > gpurun_out/e2e2c1.json 2>gpurun_out/e2e2.err; python -c "
import json; d=json.loads(open('gpurun_out/e2e2c1.json').read().strip().splitlines()[-1]); print('bench c1', d['value'], d['latency_ms'], 'e2e', d['e2e'])"
