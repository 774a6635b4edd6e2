mkdir -p gpurun_out/p
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 > gpurun_out/p/b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 > gpurun_out/p/ncu_l.log 2>&1
echo launches rc=$?
python tools/profile_run.py --iters 2 > gpurun_out/p/pr.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:conv3x3_tc_kernelILi8E' -s 1 -c 1 -o gpurun_out/p/stack_full python tools/profile_run.py --iters 2 > gpurun_out/p/ncu_full.log 2>&1
echo full rc=$?
TVS_STACK=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:conv3x3_tc_kernelILi0E' -s 20 -c 1 -o gpurun_out/p/hidden_full python tools/profile_run.py --iters 2 > gpurun_out/p/ncu_full0.log 2>&1
echo full0 rc=$?
