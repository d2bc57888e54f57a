"""Window attribution (NX_PHASE_TIMERS=2 diagnostic build): wall of the
arrival windows, and the part spent in windows where an engine ran a
structural refit."""
import os, sys
os.environ["NX_PHASE_TIMERS"] = "2"
os.environ.setdefault("NX_SO", os.path.join(os.path.dirname(os.path.abspath(__file__)), "_timers", "_nxsched.so"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2509_23384_b200 import sim, workloads as W
HZ = 1.965e9
cfgs = [W.sweep_replica(r, 1, p, 2000) for r in (10.0, 25.0, 47.5) for p in ("prism", "round_robin")]
b = sim.Batch(cfgs)
b.run()
for i, c in enumerate(cfgs):
    cy = b.phase_cycles(i)
    t0, t1 = b.timeline(i)
    print(f"rate {c['workload']['rate']:5.1f} {c['router']['policy']:12s} wall {(t1 - t0) / 1e9:.3f}s "
          f"windows {cy[14] / HZ:.3f}s of which refit windows {cy[12] / HZ:.3f}s ({cy[13]} windows) "
          f"structural(sum) {cy[6] / HZ:.3f}s events(sum) {cy[10] / HZ:.3f}s")
