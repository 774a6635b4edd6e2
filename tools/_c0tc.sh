timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python tools/ab_env.py TVS_CONV0_CUDA=1 --reps 20 2>&1 | grep -E "bitwise|default|TVS" | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv0 -c 2 python tools/profile_run.py --iters 2 2>&1 | grep -E "conv0|duration" | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv0 -c 2 python tools/profile_run.py --unshuffle 2 --iters 2 2>&1 | grep -E "conv0|duration" | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --fp32-steps 0 --fp32-fast-steps 0 > gpurun_out/c0tc.json 2>gpurun_out/c0tc.err; python -c "
import json; d=json.loads(open('gpurun_out/c0tc.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], 'share', d['roofline']['share_of_step'], 'e2e', d['e2e']['value'], 'u2', d.get('unshuffle2_variant',{}).get('value'))"
