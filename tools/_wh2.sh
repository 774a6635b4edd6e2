timeout 300 python tools/ab_env.py TVS_WIDE_PAIR=0 --wide 1 --config 5 --imgs 16 --reps 6 2>&1 | grep -E "default|TVS" | tail -2
