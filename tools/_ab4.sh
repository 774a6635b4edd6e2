mkdir -p gpurun_out/ab4
timeout 300 python tools/ab_env.py TVS_CONV_DBG=4096 --reps 20 > gpurun_out/ab4/old.log 2>&1; tail -4 gpurun_out/ab4/old.log
timeout 300 python tools/ab_env.py TVS_CONV_DBG=1 --reps 20 > gpurun_out/ab4/nowait.log 2>&1; tail -3 gpurun_out/ab4/nowait.log
timeout 300 python tools/ab_env.py TVS_CONV_DBG=4096 --config 5 --imgs 128 --reps 8 > gpurun_out/ab4/old_c5.log 2>&1; tail -4 gpurun_out/ab4/old_c5.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-steps 0 --unshuffle-steps 0 > gpurun_out/ab4/bench.json 2> gpurun_out/ab4/bench.err; tail -c 300 gpurun_out/ab4/bench.json
