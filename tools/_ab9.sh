timeout 300 python tools/ab_env.py TVS_CONV_DBG=4096 --reps 20 2>&1 | grep -E "config|default|TVS" | tail -3
timeout 300 python tools/ab_env.py TVS_CONV_DBG=4096 --config 5 --imgs 128 --reps 8 2>&1 | grep -E "default|TVS" | tail -2
