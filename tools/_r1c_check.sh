# re-entry check: full GPU suite + default bench + wide bench
mkdir -p gpurun_out/r1c
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r1c/gpu_tests.log 2>&1; tail -3 gpurun_out/r1c/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1c/bench.json 2> gpurun_out/r1c/bench.err; tail -c 600 gpurun_out/r1c/bench.json
timeout 900 python bench.py --config 5w --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/r1c/bench5w.json 2> gpurun_out/r1c/bench5w.err; tail -c 600 gpurun_out/r1c/bench5w.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1c/smoke.log 2>&1; tail -3 gpurun_out/r1c/smoke.log
