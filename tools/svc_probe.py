import os, sys
os.environ.setdefault("NX_PHASE_TIMERS", "1")
os.environ.setdefault("NX_SO", os.path.join(os.path.dirname(os.path.abspath(__file__)), "_timers", "_nxsched.so"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2509_23384_b200 import sim, workloads as W
c = W.sweep_replica(10.0, 1, "round_robin", 2000)
b = sim.Batch([c]); b.run()
cy = b.phase_cycles(0); t0, t1 = b.timeline(0); w = b.work(0)
print("wall", (t1 - t0) / 1e9, "structural(wait)", cy[6] / 1.965e9, "events", cy[10] / 1.965e9, "fits", w[5], "status", b.summaries()[0].status)
NAMES = ["merge", "route", "plan", "complete", "report", "linear", "structural", "park", "ring", "drain",
         "events", "router-idle", "final", "windows", "n_windows", "learn"]
print("  ".join(f"{n} {v / 1.965e9:.3f}" for n, v in zip(NAMES, cy) if v))
