"""Per-phase SM-cycle attribution of single replicas (latency analysis)."""
import argparse, os, sys
os.environ.setdefault("NX_PHASE_TIMERS", "1")
# the product library has no phase timers: use (and if needed build) the
# diagnostic -DNX_TIMERS build
_TIMERS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_timers", "_nxsched.so")
if "NX_SO" not in os.environ:
    if not os.path.exists(_TIMERS):
        import subprocess
        _csrc = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2509_23384_b200", "csrc")
        subprocess.run(["make", "-C", _csrc, f"OUT={_TIMERS}", f"B={os.path.dirname(_TIMERS)}/build",
                        "EXTRA=-DNX_TIMERS"], check=True, stdout=subprocess.DEVNULL)
    os.environ["NX_SO"] = _TIMERS
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_23384_b200 import sim, workloads as W
NAMES = ["select+hash", "route+admit", "plan(LENS)", "complete", "report", "linear", "structural*", "fit-tables", "refit-wait", "fit-pass", "fit-total", "cheap-sum", "stage", "fit-solve", "exact-fit", "solve5"]
ap = argparse.ArgumentParser()
ap.add_argument("--requests", type=int, default=2000)
a = ap.parse_args()
cfgs = [W.sweep_replica(r, 1, p, a.requests) for r in (10.0, 25.0, 47.5) for p in ("prism", "round_robin")]
b = sim.Batch(cfgs)
b.run()
print(f"kernel {b.kernel_ms():.1f} ms for {len(cfgs)} replicas")
for i, c in enumerate(cfgs):
    cyc = b.phase_cycles(i); tot = sum(cyc[:9]) - cyc[6] - cyc[7]  # refit-warp phases overlap
    s = b.summaries()[i]; w = b.work(i)
    print(f"rate {c['workload']['rate']:5.1f} {c['router']['policy']:12s} events {s.events:7d} dec {s.decisions:7d} "
          f"total {tot/1.9e9:6.3f}s  cyc/event {tot/max(1,s.events):7.0f}  steps {w[0]} fits {w[5]}")
    print("    " + "  ".join(f"{n} {100*v/tot:4.1f}%" for n, v in zip(NAMES, cyc)))
