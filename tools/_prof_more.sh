mkdir -p gpurun_out/pm
P="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
python tools/profile_run.py --iters 2 > gpurun_out/pm/a.log 2>&1 && \
timeout 600 $P -k 'regex:conv0_kernel|conv3x3_tc_kernelILi1E' -s 2 -c 2 -o gpurun_out/pm/edge python tools/profile_run.py --iters 2 > gpurun_out/pm/edge.log 2>&1; echo edge $?
python tools/profile_run.py --config 5w --batch 16 --iters 1 > gpurun_out/pm/w.log 2>&1 && \
timeout 900 $P -k 'regex:conv3x3_tc_kernelILi(5|9|10)E' -s 0 -c 3 -o gpurun_out/pm/wide python tools/profile_run.py --config 5w --batch 16 --iters 1 > gpurun_out/pm/wide.log 2>&1; echo wide $?
timeout 600 $P -k 'regex:conv3x3_tc_kernelILi9E' -s 12 -c 1 -o gpurun_out/pm/wide9 python tools/profile_run.py --config 5w --batch 16 --iters 1 > gpurun_out/pm/wide9.log 2>&1; echo wide9 $?
python tools/profile_run.py --unshuffle 2 --iters 2 > gpurun_out/pm/u.log 2>&1 && \
timeout 600 $P -k 'regex:conv0_unshuffle|conv3x3_tc_kernelILi7E' -s 2 -c 2 -o gpurun_out/pm/unshuf python tools/profile_run.py --unshuffle 2 --iters 2 > gpurun_out/pm/unshuf.log 2>&1; echo unshuf $?
