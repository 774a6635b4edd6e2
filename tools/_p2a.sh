timeout 120 python tools/ab_env.py TVS_PAIR2=1 TVS_STACK=0 --imgs 8 --reps 10 > gpurun_out/p2a.log 2>&1
echo "rc=$?"; tail -12 gpurun_out/p2a.log
