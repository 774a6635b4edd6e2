"""Aggregate the last training step of an ncu launch list made with
    ncu --metrics gpu__time_duration.sum --clock-control none -c 2400 --csv --log-file X python tools/bench_train.py --steps 1 --cpu-steps 1
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
rows = rows[1:]
start = [i for i, r in enumerate(rows) if "train_pack_hidden_kernel" in r[ki]][-1]
agg, tot = collections.OrderedDict(), 0.0
for r in rows[start:]:
    k, v = r[ki][:60], float(r[vi])
    tot += v
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"{c:5d} {v / 1e3:9.1f} us  {v / c / 1e3:7.1f} us/launch  {k}")
print(f"total {tot / 1e3:.1f} us in {len(rows) - start} launches")
