timeout 300 python tools/ab_env.py TVS_WIDE_HALVES=0 --wide 1 --config 5 --imgs 16 --reps 6 2>&1 | grep -E "bitwise|default|TVS" | tail -8
timeout 900 python -m pytest tests -q -m gpu -k "wide" 2>&1 | tail -2
