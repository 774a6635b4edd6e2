mkdir -p gpurun_out/val2
for c in 1 3 4 5 5w; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/val2/bench_c$c.json 2> gpurun_out/val2/bench_c$c.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/val2/ref.json 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 > gpurun_out/val2/b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/val2/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 > gpurun_out/val2/ncu_l.log 2>&1
for f in gpurun_out/val2/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('impl','ours'), d.get('value'), d.get('unit'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'), d.get('latency_ms'))"; done
