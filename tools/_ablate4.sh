for v in "TVS_STACK=0 TVS_CONV_DBG=48" "TVS_STACK=0 TVS_CONV_DBG=560" "TVS_STACK=0 TVS_CONV_DBG=1072" "TVS_STACK=0 TVS_CONV_DBG=1584" "TVS_STACK=0" "TVS_STACK=0 TVS_CONV_DBG=1536" "TVS_STACK=1" "TVS_STACK=1 TVS_CONV_DBG=1536"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$v', d['value'], d['ms_per_step'], r['avg_launch_ms'], r['launches_timed'], d['clocks']['sm_mhz'])"
done
