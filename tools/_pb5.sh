for d in 0 1; do echo "== stack pb dbg=$d"; timeout 300 python tools/ab_env.py TVS_PB=1 TVS_CONV_DBG=$d --reps 10 2>&1 | grep -E "TVS|default" | tail -2; done
