mkdir -p gpurun_out/sb
for i in 1 2; do
for v in "TVS_STACK=0" "TVS_STACK=1" "TVS_STACK=1 TVS_STACK_SKEW=2"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['clocks'])"
done; done
