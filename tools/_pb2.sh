for d in 1 3; do echo "== stack pb dbg=$d"; timeout 300 python tools/ab_env.py TVS_PB=1 TVS_CONV_DBG=$d --reps 10 2>&1 | grep -E "default|TVS" | tail -2; done
