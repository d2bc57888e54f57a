"""Per-phase cycles per event: the same replicas alone on an SM vs. inside the
full bench-shard launch (where does co-residency / load slow the event loop?)."""
import os, sys
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
from collections import defaultdict
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_23384_b200 import sim, workloads as W
NAMES = ["select+hash", "route+admit", "plan", "complete", "report", "linear", "structural*", "fit-tables",
         "refit-wait", "fit-pass", "fit-total", "less_scaled", "stage", "fit-solve", "base-err", "solve5"]

def per_event(b, idx):
    acc = [0.0] * 16; ev = 0
    for i in idx:
        cyc = b.phase_cycles(i)
        for k in range(16): acc[k] += cyc[k]
        ev += b.summaries()[i].events
    return [a / max(1, ev) for a in acc], ev

cfgs = W.sweep_configs(n_replicas=512, n=2000)
full = sim.Batch(cfgs, host_threads=os.cpu_count()); full.run()
print(f"full shard: kernel {full.kernel_ms():.1f} ms")
by = defaultdict(list)
for i, c in enumerate(cfgs):
    by[(c["workload"]["rate"], c["router"]["policy"])].append(i)
pick = [(10.0, "prism"), (10.0, "least_loaded"), (25.0, "prism"), (47.5, "prism"), (47.5, "latency_based")]
iso_idx = [by[k][0] for k in pick]
iso = sim.Batch([cfgs[i] for i in iso_idx]); iso.run()
print("cycles/event          " + " ".join(f"{n[:10]:>10s}" for n in NAMES[:11]))
for j, k in enumerate(pick):
    a, ev = per_event(iso, [j])
    f, _ = per_event(full, [iso_idx[j]])
    g, _ = per_event(full, by[k])
    for tag, v in (("alone", a), ("in shard", f), ("shard avg", g)):
        print(f"{k[0]:5.1f} {k[1][:12]:12s} {tag:9s} " + " ".join(f"{x:10.0f}" for x in v[:11]))
print("linear refits (alone runs): count, cycles per refit, learner counters summed")
for j, k in enumerate(pick):
    w = iso.work(j); cyc = iso.phase_cycles(j); nl = max(1, w[3] // 64)
    cnt = [0] * 7
    for e in range(len(cfgs[iso_idx[j]]["engines"])):
        for q, v in enumerate(iso.learner(j, e)[2]): cnt[q] += v
    print(f"{k[0]:5.1f} {k[1][:12]:12s} n {nl:6d} cyc {cyc[5]/nl:8.0f} cnt {cnt}")
