mkdir -p gpurun_out
python tools/bench_producer.py --images 148 --size 64 --steps 4 --cpu-images 0 > gpurun_out/pb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tvflow_cluster -s 1 -c 1 -o gpurun_out/tvflow_full2 python tools/bench_producer.py --images 148 --size 64 --steps 4 --cpu-images 0 > gpurun_out/ncu_tv.log 2>&1
tail -1 gpurun_out/pb.log; tail -2 gpurun_out/ncu_tv.log
