mkdir -p gpurun_out/ab1
timeout 600 python tools/ab_env.py TVS_DIRECT=1 > gpurun_out/ab1/direct.log 2>&1; tail -4 gpurun_out/ab1/direct.log
timeout 600 python tools/ab_env.py TVS_DIRECT=1 TVS_STACK=0 > gpurun_out/ab1/direct_nostack.log 2>&1; tail -4 gpurun_out/ab1/direct_nostack.log
timeout 600 python tools/ab_env.py TVS_STACK=0 > gpurun_out/ab1/nostack.log 2>&1; tail -3 gpurun_out/ab1/nostack.log
timeout 600 python tools/ab_env.py TVS_DIRECT=1 --config 5 --imgs 128 --reps 8 > gpurun_out/ab1/direct_c5.log 2>&1; tail -3 gpurun_out/ab1/direct_c5.log
