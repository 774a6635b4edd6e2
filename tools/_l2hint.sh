for cfg in "0 1" "1 1" "3 1" "2 1" "1 2" "3 2" "1 4" "3 4"; do set -- $cfg
  r=$(TVS_L2_HINTS=$1 TVS_REVERSE_SUB=$2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])")
  echo "hints=$1 rev=$2 -> $r"
done
