mkdir -p gpurun_out/ab6
timeout 300 python tools/ab_env.py TVS_CONV_DBG=16384 --reps 20 > gpurun_out/ab6/static.log 2>&1; grep -E "bitwise|default|TVS|AB_" gpurun_out/ab6/static.log | tail -5
timeout 300 python tools/ab_env.py TVS_CONV_DBG=16384 --config 5 --imgs 128 --reps 8 > gpurun_out/ab6/static_c5.log 2>&1; grep -E "default|TVS|AB_" gpurun_out/ab6/static_c5.log | tail -3
timeout 600 python -m pytest tests -q -m gpu -k "stack or configs" > gpurun_out/ab6/tests.log 2>&1; tail -2 gpurun_out/ab6/tests.log
