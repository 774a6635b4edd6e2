mkdir -p gpurun_out/val6
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 5 --fp32-steps 0 > gpurun_out/val6/bench_c$c.json 2> gpurun_out/val6/bench_c$c.err; done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/val6/bench_c2.json 2> gpurun_out/val6/bench_c2.err
for f in gpurun_out/val6/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('kernel','')[:30], (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'), d.get('latency_ms'), d.get('fp32_mode',{}).get('value'), d.get('unshuffle2_variant',{}).get('value'))"; done
