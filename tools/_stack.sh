mkdir -p gpurun_out/s
timeout 300 python tools/stack_check.py 64 1 2 3 4 > gpurun_out/s/stack.log 2>&1; echo rc=$?; cat gpurun_out/s/stack.log | tail -20
