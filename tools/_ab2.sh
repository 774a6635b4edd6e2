mkdir -p gpurun_out/ab2
for d in 4096 8192 12288; do
timeout 600 python tools/ab_env.py TVS_DIRECT=1 TVS_CONV_DBG=$d > gpurun_out/ab2/d$d.log 2>&1; tail -4 gpurun_out/ab2/d$d.log
done
