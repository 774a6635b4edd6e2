timeout 300 python tools/ab_env.py TVS_STACK=1 --reps 20 2>&1 | grep -E "default" | tail -1 | sed "s/^/g3s6 c2: /"
timeout 300 python tools/ab_env.py TVS_STACK=1 --config 5 --imgs 128 --reps 8 2>&1 | grep -E "default" | tail -1 | sed "s/^/g3s6 c5: /"
cp paper_2006_10004_b200/libtvsb200_g4s5.so paper_2006_10004_b200/libtvsb200.so
timeout 300 python tools/ab_env.py TVS_STACK=1 --reps 20 2>&1 | grep -E "default|AB_" | tail -2 | sed "s/^/g4s5 c2: /"
timeout 300 python tools/ab_env.py TVS_STACK=1 --config 5 --imgs 128 --reps 8 2>&1 | grep -E "default" | tail -1 | sed "s/^/g4s5 c5: /"
