"""Phase seconds of one RR replica alone vs. 148 copies (diagnostic build)."""
import os, sys
os.environ.setdefault("NX_PHASE_TIMERS", "1")
os.environ.setdefault("NX_SO", os.path.join(os.path.dirname(os.path.abspath(__file__)), "_timers", "_nxsched.so"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2509_23384_b200 import sim, workloads as W
NAMES = ["merge", "route", "plan", "complete", "report", "linear", "structural", "park", "ring", "drain",
         "events", "router-idle", "final", "windows", "n_windows", "learn"]
c = W.sweep_replica(10.0, 1, "round_robin", 2000)
for n in (1, 148):
    b = sim.Batch([c] * n, host_threads=os.cpu_count())
    b.run()
    cy = b.phase_cycles(0)
    t0, t1 = b.timeline(0)
    print(f"copies {n}: wall {(t1 - t0) / 1e9:.3f}s  " + "  ".join(f"{k} {v / 1.965e9:.3f}" for k, v in zip(NAMES, cy) if v), flush=True)
    b.close()
