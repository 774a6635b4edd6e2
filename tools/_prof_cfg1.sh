mkdir -p gpurun_out
python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 > gpurun_out/c1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -c 60 --csv --log-file gpurun_out/c1_launches.csv python bench.py --config 1 --steps 1 --warmup 1 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 > gpurun_out/c1_ncu.log 2>&1
tail -1 gpurun_out/c1.log | cut -c1-300
