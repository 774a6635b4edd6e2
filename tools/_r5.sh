timeout 300 python tools/ab_env.py TVS_STACK=0 --precision fp32 --reps 10 2>&1 | grep -E "default|TVS" | tail -2
timeout 900 python -m pytest tests -q -m gpu -k "fp32 or golden or configs or wide or stack" 2>&1 | tail -2
