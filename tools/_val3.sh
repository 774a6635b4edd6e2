mkdir -p gpurun_out/val3
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 900 python bench.py --config 5w --steps 3 --warmup 3 --cpu-seconds 5 --fp32-steps 0 > gpurun_out/val3/bench_c5w.json 2> gpurun_out/val3/bench_c5w.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/val3/bench_c2.json 2> gpurun_out/val3/bench_c2.err
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for f in gpurun_out/val3/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['roofline']['kernel'][:45], d['roofline']['frac'], d['clocks'], d.get('fp32_mode',{}).get('value'), d.get('unshuffle2_variant',{}).get('value'))"; done
