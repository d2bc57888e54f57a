"""Per-replica phase attribution of the engine-parallel simulation kernel
(diagnostic -DNX_TIMERS build): wall time per replica, where the router warp
and the engine warps spend their cycles, and a bench-shard timeline."""
import argparse, os, sys
os.environ.setdefault("NX_PHASE_TIMERS", "1")
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

NAMES = ["merge", "route", "plan", "complete", "report", "linear", "structural", "park", "ring", "drain",
         "events", "router-idle", "final", "windows", "n_windows", "learn"]
ap = argparse.ArgumentParser()
ap.add_argument("--requests", type=int, default=2000)
ap.add_argument("--shard", type=int, default=0, help="also time a bench shard of this many replicas")
a = ap.parse_args()
HZ = 1.965e9
cfgs = [W.sweep_replica(r, 1, p, a.requests) for r in (10.0, 25.0, 47.5) for p in ("prism", "round_robin")]
b = sim.Batch(cfgs)
b.run()
print(f"kernel {b.kernel_ms():.1f} ms for {len(cfgs)} replicas")
for i, c in enumerate(cfgs):
    cyc = b.phase_cycles(i)
    s = b.summaries()[i]
    w = b.work(i)
    t0, t1 = b.timeline(i)
    wall = (t1 - t0) / 1e9
    print(f"rate {c['workload']['rate']:5.1f} {c['router']['policy']:12s} wall {wall:6.3f}s events {s.events:7d} "
          f"dec {s.decisions:7d} ns/event {1e9 * wall / max(1, s.events):6.0f} steps {w[0]} fits {w[5]} windows {cyc[14]}")
    router = {n: cyc[k] / HZ for k, n in enumerate(NAMES) if n in ("merge", "route", "router-idle", "final", "windows")}
    eng = {n: cyc[k] / HZ for k, n in enumerate(NAMES) if n in ("events", "plan", "complete", "report", "linear",
                                                               "structural", "learn", "park", "ring", "drain")}
    print("    router s: " + "  ".join(f"{n} {v:6.3f}" for n, v in router.items()))
    print("    engine-warp s (sum over warps): " + "  ".join(f"{n} {v:6.3f}" for n, v in eng.items()))
if a.shard:
    cfgs = W.sweep_configs(n_replicas=a.shard, n=a.requests)
    b = sim.Batch(cfgs, host_threads=os.cpu_count())
    b.run()
    tl = [b.timeline(r) for r in range(len(cfgs))]
    t0 = min(x[0] for x in tl)
    spans = [((x[0] - t0) / 1e6, (x[1] - t0) / 1e6) for x in tl]
    end = max(e for _, e in spans)
    print(f"shard {a.shard}: kernel {b.kernel_ms():.1f} ms; sum of replica durations "
          f"{sum(e - s for s, e in spans):.0f} ms over {end:.0f} ms")
    from collections import defaultdict
    by = defaultdict(list)
    for r, c in enumerate(cfgs):
        by[c["workload"]["rate"]].append(spans[r][1] - spans[r][0])
    for rate in sorted(by):
        v = sorted(by[rate])
        print(f"  rate {rate:5.1f}: n {len(v)} dur ms min {v[0]:.1f} med {v[len(v)//2]:.1f} max {v[-1]:.1f}")
