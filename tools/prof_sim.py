"""Profiling driver: one launch of the lockstep kernel over a small shard."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_23384_b200 import sim, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--replicas", type=int, default=8)
ap.add_argument("--requests", type=int, default=400)
ap.add_argument("--launches", type=int, default=1)
a = ap.parse_args()
cfgs = W.sweep_configs(a.replicas, a.requests)
b = sim.Batch(cfgs)
b.upload()
for _ in range(a.launches):
    b.launch(); b.synchronize()
    print(f"kernel {b.kernel_ms():.1f} ms")
b.download(); b.synchronize()
s = b.summaries()
print("decisions", sum(x.decisions for x in s), "status", set(x.status for x in s))
