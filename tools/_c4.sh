for mb in 2048 8192; do TVS_CHUNK_MB=$mb timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --fp32-fast-steps 0 --unshuffle-steps 0 --fp32-steps 0 --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('chunk $mb', d['value'], d['roofline']['kernel'][:30], d['clocks'])"; done
