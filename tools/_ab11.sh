for i in 1 2; do
timeout 300 python tools/ab_env.py TVS_CONV_DBG=8192 --reps 40 2>&1 | grep -E "default|TVS" | tail -2
timeout 300 python tools/ab_env.py TVS_CONV_DBG=8192 --config 5 --imgs 128 --reps 12 2>&1 | grep -E "default|TVS" | tail -2
done
