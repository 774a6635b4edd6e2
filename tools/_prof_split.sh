mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --fp32-steps 0 --no-cpu-baseline > gpurun_out/pbs.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:conv3x3_tc_kernelILi3E' -s 3 -c 1 -o gpurun_out/split_full python bench.py --steps 2 --warmup 1 --fp32-steps 0 --no-cpu-baseline --fp32-fast-steps 1 > gpurun_out/ncu_split.log 2>&1
tail -2 gpurun_out/ncu_split.log
