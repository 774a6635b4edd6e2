for v in 0 8 24 32; do echo "seg=$v"; timeout 300 python tools/ab_env.py TVS_SPLIT_SEG=$v --precision fp32 --reps 10 2>&1 | grep -E "bitwise|default|TVS|AB_" | tail -4; done
