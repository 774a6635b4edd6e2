timeout 300 python tools/ab_env.py TVS_CONV_DBG=8192 --reps 20 2>&1 | grep -E "bitwise|default|TVS|AB_" | tail -9
timeout 300 python tools/ab_env.py TVS_CONV_DBG=8192 --config 5 --imgs 128 --reps 8 2>&1 | grep -E "default|TVS" | tail -2
