timeout 300 env TVS_CONV0_TC=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv0 -c 2 python tools/profile_run.py --iters 2 2>&1 | grep -E "duration" | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv0 -c 2 python tools/profile_run.py --unshuffle 2 --iters 2 2>&1 | grep -E "duration" | tail -2
timeout 900 python -m pytest tests -q -m gpu -x -k "conv0 or unshuffle or golden" 2>&1 | tail -2
