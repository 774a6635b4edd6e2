for d in 49 1585 65 ; do timeout 300 python tools/ab_env.py TVS_CONV_DBG=$d --reps 20 2>&1 | grep -E "TVS" | tail -1 | sed "s/^/dbg=$d: /"; done
