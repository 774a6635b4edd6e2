set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/r2_smi.txt
for c in 2 1 3 5 5w 4; do
  timeout 900 python bench.py --config $c > gpurun_out/r2_bench_cfg$c.json 2> gpurun_out/r2_bench_cfg$c.err
done
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --fp32-fast-steps 0 --fp32-steps 0 --unshuffle-steps 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel -c 2 -o gpurun_out/r2_stack_full python bench.py --steps 1 --warmup 3 --fp32-fast-steps 0 --fp32-steps 0 --unshuffle-steps 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2_ncu_full.log 2>&1
python tools/bench_train.py > gpurun_out/r2_train_step_128.json 2> gpurun_out/r2_train_step_128.err
python tools/bench_train.py --size 64 > gpurun_out/r2_train_step_64.json 2> gpurun_out/r2_train_step_64.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2400 --csv --log-file gpurun_out/r2_launches_train_step.csv python tools/bench_train.py --steps 1 --cpu-steps 1 > gpurun_out/r2_ncu_train.log 2>&1
