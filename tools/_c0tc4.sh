timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/c0tc4.json 2>gpurun_out/c0tc4.err; python -c "
import json; d=json.loads(open('gpurun_out/c0tc4.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], 'frac', d['roofline']['frac'], 'share', d['roofline']['share_of_step'], 'e2e', d['e2e']['value'], 'u2', d.get('unshuffle2_variant',{}).get('value'), 'fp32', d.get('fp32_mode',{}).get('value'), d['clocks'])"
