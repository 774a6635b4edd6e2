timeout 300 python -m pytest tests -q -m gpu -k "fp32 or golden or configs" 2>&1 | tail -1
timeout 300 python tools/ab_env.py TVS_STACK=0 --precision fp32 --reps 10 2>&1 | grep -E "default|TVS" | tail -2
