for v in "TVS_STACK=1" "TVS_STACK=1 TVS_L2_HINTS=2" "TVS_STACK=1 TVS_L2_HINTS=1" "TVS_STACK=1 TVS_L2_HINTS=3" "TVS_STACK=0" "TVS_STACK=1"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$v', d['value'], d['ms_per_step'], r['avg_launch_ms'], r['launches_timed'], d['clocks']['sm_mhz'], r['kernel'])"
done
mkdir -p gpurun_out/sl
for h in 0 2; do
TVS_STACK=1 TVS_L2_HINTS=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --kernel-name-base mangled -k 'regex:conv3x3_tc_kernelILi8E' -s 1 -c 1 --csv python tools/profile_run.py --iters 2 > gpurun_out/sl/ncu_h$h.csv 2>&1; grep -E "dram|time_dur|hit_rate|tensor" gpurun_out/sl/ncu_h$h.csv | cut -d, -f12- 
done
