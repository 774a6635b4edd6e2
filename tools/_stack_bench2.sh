for c in 5 4 3; do
for v in "TVS_STACK=0" "TVS_STACK=1 TVS_CHUNK_MB=8192" "TVS_STACK=0 TVS_CHUNK_MB=8192"; do
  env $v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$c $v', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['clocks'])"
done; done
