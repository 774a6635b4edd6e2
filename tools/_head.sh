timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:conv3x3_tc_kernelILi1E -c 2 python tools/profile_run.py --iters 2 2>&1 | grep -E "duration" | tail -2
timeout 600 python -m pytest tests -q -m gpu -x -k "golden or configs or ragged or window" 2>&1 | tail -1
