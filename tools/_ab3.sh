mkdir -p gpurun_out/ab3
for d in 1 17 33 257 65 1537 49 161 2048; do
echo "dbg=$d"; timeout 300 python tools/ab_env.py TVS_CONV_DBG=$d --reps 10 > gpurun_out/ab3/d$d.log 2>&1; tail -2 gpurun_out/ab3/d$d.log | head -1
done
