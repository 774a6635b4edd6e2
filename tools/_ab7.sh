mkdir -p gpurun_out/ab7
echo "== bitwise: forced stack, 3 bands vs per-layer"; timeout 300 python tools/ab_env.py TVS_STACK=1 TVS_STACK_BANDS=3 --imgs 16 --reps 5 > gpurun_out/ab7/b3.log 2>&1; grep -E "bitwise|default|TVS|AB_" gpurun_out/ab7/b3.log | tail -9
echo "== e2e-size sub-batch 16 imgs: auto stack (3 bands) vs per-layer"; timeout 300 python tools/ab_env.py TVS_STACK=0 --imgs 16 --reps 20 > gpurun_out/ab7/s16.log 2>&1; grep -E "default|TVS|AB_" gpurun_out/ab7/s16.log | tail -3
echo "== config 3: forced stack (auto bands) vs per-layer"; timeout 300 python tools/ab_env.py TVS_STACK=1 --config 3 --imgs 1 --reps 20 > gpurun_out/ab7/c3.log 2>&1; grep -E "default|TVS|AB_" gpurun_out/ab7/c3.log | tail -3
echo "== config 4 (2 planes): auto stack (8 bands) vs per-layer"; timeout 300 python tools/ab_env.py TVS_STACK=0 --config 4 --imgs 2 --reps 6 > gpurun_out/ab7/c4.log 2>&1; grep -E "default|TVS|AB_" gpurun_out/ab7/c4.log | tail -3
echo "== config 2 sanity"; timeout 300 python tools/ab_env.py TVS_STACK=0 --reps 10 > gpurun_out/ab7/c2.log 2>&1; grep -E "default|TVS|AB_" gpurun_out/ab7/c2.log | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-steps 0 --unshuffle-steps 0 --fp32-fast-steps 0 > gpurun_out/ab7/bench.json 2> gpurun_out/ab7/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/ab7/bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], 'e2e', d['e2e'], d['clocks'])"
