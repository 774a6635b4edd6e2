mkdir -p gpurun_out/p2
python tools/profile_run.py --iters 2 > gpurun_out/p2/pr.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:conv3x3_tc_kernelILi8E' -s 1 -c 1 -o gpurun_out/p2/stack_full python tools/profile_run.py --iters 2 > gpurun_out/p2/ncu_full.log 2>&1
echo full rc=$?
