mkdir -p gpurun_out/t
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t/gpu_tests.log 2>&1; tail -3 gpurun_out/t/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/t/bench.json 2> gpurun_out/t/bench.err; tail -c 1500 gpurun_out/t/bench.json
