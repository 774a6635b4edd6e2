timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/val4_c2.json 2> gpurun_out/val4_c2.err; python -c "
import json; d=json.loads(open('gpurun_out/val4_c2.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], d['clocks'])"
