mkdir -p gpurun_out/v
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/v/gpu_tests.log 2>&1; tail -3 gpurun_out/v/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/v/bench.json 2> gpurun_out/v/bench.err; tail -c 600 gpurun_out/v/bench.json
TVS_PAIR=1 timeout 300 python tools/pair_check.py 64 256 > gpurun_out/v/pair.log 2>&1; tail -5 gpurun_out/v/pair.log
