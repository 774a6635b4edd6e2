mkdir -p gpurun_out/s
timeout 300 python tools/stack_check.py 64 1 8 skew4 skew2 skew1 > gpurun_out/s/stack.log 2>&1; echo rc=$?; tail -12 gpurun_out/s/stack.log
#TVS_STACK=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:conv3x3_tc_kernelILi8E' -s 1 -c 1 -o gpurun_out/s/stack_full python tools/profile_run.py --iters 2 > gpurun_out/s/ncu.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/s/ncu.log
