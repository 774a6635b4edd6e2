timeout 300 python tools/ab_env.py TVS_WIDE_HALVES=0 --wide 1 --config 5 --imgs 16 --reps 6 2>&1 | grep -E "bitwise|default|TVS" | tail -8
for P in 12 0; do timeout 300 python tools/ab_env.py TVS_WIDE_HALVES=0 TVS_WIDE_PAIR=$P --wide 1 --config 5 --imgs 16 --reps 6 2>&1 | grep -E "default|TVS" | tail -2; done
timeout 900 python -m pytest tests -q -m gpu -k "wide" 2>&1 | tail -2
