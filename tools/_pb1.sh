echo "== stack: pb vs ring"; timeout 300 python tools/ab_env.py TVS_PB=1 --reps 20 2>&1 | grep -E "bitwise|default|TVS|AB_|Error|error" | tail -9
echo "== per-layer: pb vs ring"; timeout 300 python tools/ab_env.py TVS_PB=1 TVS_STACK=0 --reps 20 2>&1 | grep -E "default|TVS|AB_" | tail -3
timeout 300 python tools/stack_check.py 2>&1 | tail -3
