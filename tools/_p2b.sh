for n in 8 32 64; do timeout 120 python tools/ab_env.py TVS_PAIR2=1 TVS_STACK=0 --imgs $n --reps 10 2>&1 | grep -E "default|TVS" | tail -2 | sed "s/^/s4g2 n=$n: /"; done
cp paper_2006_10004_b200/libtvsb200_s3g3.so paper_2006_10004_b200/libtvsb200.so
for n in 8 32 64; do timeout 120 python tools/ab_env.py TVS_PAIR2=1 TVS_STACK=0 --imgs $n --reps 10 2>&1 | grep -E "TVS|AB_" | tail -2 | sed "s/^/s3g3 n=$n: /"; done
