mkdir -p gpurun_out/ab5
for d in 131072 262144 524288 786432; do
echo "dbg=$d"; timeout 300 python tools/ab_env.py TVS_CONV_DBG=$d --reps 16 > gpurun_out/ab5/d$d.log 2>&1; grep -E "default|TVS|AB_" gpurun_out/ab5/d$d.log | tail -3
done
