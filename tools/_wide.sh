timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "wide" 2>&1 | tail -3
for P in 24 12 0; do
  TVS_WIDE_PAIR=$P timeout 900 python bench.py --config 5w --steps 3 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('P=$P', d['value'], d['ms_per_step'], r['avg_launch_ms'], r['achieved'], d['clocks'])"
done
