timeout 300 python -m pytest tests -q -m gpu -k "host or cpu_tensors or export" 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-steps 0 --unshuffle-steps 0 --fp32-fast-steps 0 --e2e-steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], 'e2e', d['e2e']['value'])"; done
