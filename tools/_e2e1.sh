timeout 300 python tools/host_chunk_sweep.py
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-steps 0 --unshuffle-steps 0 --fp32-fast-steps 0 > gpurun_out/e2e1.json 2>gpurun_out/e2e1.err; python -c "
import json; d=json.loads(open('gpurun_out/e2e1.json').read().strip().splitlines()[-1]); print('bench', d['value'], 'e2e', d['e2e'])"
