for nb in 1 4 8 16 32; do echo "bands=$nb"; timeout 300 python tools/ab_env.py TVS_STACK=1 TVS_STACK_BANDS=$nb --config 1 --imgs 1 --reps 30 2>&1 | grep -E "config|default|TVS" | tail -3; done
