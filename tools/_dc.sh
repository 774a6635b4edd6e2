timeout 300 python tools/ab_env.py TVS_DISCARD_L2=1 --reps 30 2>&1 | grep -E "bitwise|default|TVS|AB_" | tail -8
timeout 300 python tools/ab_env.py TVS_DISCARD_L2=1 --config 5 --imgs 128 --reps 10 2>&1 | grep -E "default|TVS" | tail -2
TVS_DISCARD_L2=1 timeout 120 python tools/mma_cycles.py 2 64 0
timeout 120 python tools/mma_cycles.py 2 64 0
TVS_DISCARD_L2=1 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --kernel-name-base mangled -k regex:ILi8E -c 1 python tools/profile_run.py --iters 1 2>&1 | grep -E "dram|duration" | tail -3
