timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:conv3x3_tc_kernelILi1E -c 2 python tools/profile_run.py --iters 2 2>&1 | grep -E "duration" | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:conv3x3_tc_kernelILi4E -c 2 python tools/profile_run.py --iters 2 --precision fp32 2>&1 | grep -E "duration" | tail -2
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
