"""Bench-shard timeline by router policy and rate (product build)."""
import os, sys
from collections import defaultdict
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench
from paper_2509_23384_b200 import sim
cfgs = bench.shard_configs(0, 512, 2000)
b = sim.Batch(cfgs, host_threads=os.cpu_count())
b.run()
tl = [b.timeline(r) for r in range(len(cfgs))]
t0 = min(x[0] for x in tl)
print(f"kernel {b.kernel_ms():.1f} ms")
by = defaultdict(list)
for r, c in enumerate(cfgs):
    by[(c["router"]["policy"], c["workload"]["rate"])].append(((tl[r][1] - tl[r][0]) / 1e6, (tl[r][0] - t0) / 1e6))
for pol in sorted({k[0] for k in by}):
    row = []
    for rate in (10.0, 20.0, 30.0, 47.5):
        v = by.get((pol, rate), [])
        if v:
            row.append(f"r{rate:g}: {sum(x[0] for x in v) / len(v):6.1f}ms")
    tot = sum(x[0] for k, v in by.items() if k[0] == pol for x in v)
    print(f"{pol:14s} sum {tot:8.0f} ms  " + "  ".join(row))
ends = sorted((x[1] - t0) / 1e6 for x in tl)
print("finish quantiles ms:", " ".join(f"{ends[int(q * (len(ends) - 1))]:.0f}" for q in (0.5, 0.9, 0.99, 1.0)))
