"""Structural-refit internals (NX_PHASE_TIMERS=3 diagnostic build): where a
refit's cycles go (tables, passes, cheap sums, staging, solve, exact fit)."""
import os, sys
os.environ["NX_PHASE_TIMERS"] = "3"
os.environ.setdefault("NX_SO", os.path.join(os.path.dirname(os.path.abspath(__file__)), "_timers", "_nxsched.so"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2509_23384_b200 import sim, workloads as W
HZ = 1.965e9
cfgs = [W.sweep_replica(r, 1, p, 2000) for r in (10.0, 47.5) for p in ("prism",)]
b = sim.Batch(cfgs)
b.run()
names = {8: "tables", 9: "pass", 10: "gauged(total)", 11: "cheap-sum", 12: "stage", 13: "finish(solve+ridge)",
         14: "exact-fit", 15: "solve5"}
for i, c in enumerate(cfgs):
    cy = b.phase_cycles(i)
    w = b.work(i)
    print(f"rate {c['workload']['rate']}: structural {cy[6] / HZ:.3f}s fits {w[5]} linear {cy[5] / HZ:.3f}s")
    print("   " + "  ".join(f"{n} {cy[k] / HZ:.3f}" for k, n in names.items()))
