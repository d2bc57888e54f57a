"""Per-replica device timeline of one bench-shard launch (co-residency study):
how long each replica took under load vs. its event count."""
import argparse, os, sys
from collections import defaultdict
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_23384_b200 import sim, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--replicas", type=int, default=512)
ap.add_argument("--requests", type=int, default=2000)
a = ap.parse_args()
cfgs = W.sweep_configs(n_replicas=a.replicas, n=a.requests)
b = sim.Batch(cfgs, host_threads=os.cpu_count())
b.run()
print(f"replicas {a.replicas}: kernel {b.kernel_ms():.1f} ms")
s = b.summaries()
tl = [b.timeline(r) for r in range(len(cfgs))]
t0 = min(x[0] for x in tl)
by = defaultdict(list)
for r, c in enumerate(cfgs):
    by[c["workload"]["rate"]].append(((tl[r][1] - tl[r][0]) / 1e6, (tl[r][0] - t0) / 1e6, s[r].events))
for rate in sorted(by):
    v = by[rate]
    ms = sorted(x[0] for x in v)
    ev = sum(x[2] for x in v) / len(v)
    st = max(x[1] for x in v)
    print(f"rate {rate:5.1f}: n {len(v):3d} dur ms min {ms[0]:7.1f} med {ms[len(ms)//2]:7.1f} max {ms[-1]:7.1f}  "
          f"events {ev:8.0f}  ns/event {1e6*ms[len(ms)//2]/ev:6.0f}  latest start {st:7.1f}")
# occupancy of the launch over time: replicas in flight at 20 instants
spans = [((x[0] - t0) / 1e6, (x[1] - t0) / 1e6) for x in tl]
end = max(e for _, e in spans)
print(f"sum of replica durations {sum(e - b for b, e in spans):.0f} ms over {end:.0f} ms")
print("in flight:", " ".join(str(sum(1 for b_, e_ in spans if b_ <= end * k / 20 < e_)) for k in range(20)))
ends = sorted(e for _, e in spans)
print("finish quantiles ms:", " ".join(f"{ends[int(q * (len(ends) - 1))]:.0f}" for q in (0.25, 0.5, 0.75, 0.9, 0.99, 1.0)))
