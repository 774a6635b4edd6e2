timeout 300 python tools/ab_env.py TVS_CONV_DBG=262144 --reps 30 2>&1 | grep -E "bitwise|default|TVS|AB_" | tail -8
timeout 300 python tools/ab_env.py TVS_CONV_DBG=262144 --config 5 --imgs 128 --reps 10 2>&1 | grep -E "default|TVS" | tail -2
timeout 300 python tools/ab_env.py TVS_CONV_DBG=262144 TVS_STACK=0 --reps 20 2>&1 | grep -E "default|TVS|AB_" | tail -3
