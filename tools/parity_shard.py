"""Whole bench shard (512 replicas of the 4096-replica sweep) on the device
vs the compiled reference (oracle/_ref) on the host: event hash (every
routing choice, batch composition, token budget and event time) and decision
count per replica."""
import os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from oracle_lib import Ref
from paper_2509_23384_b200 import sim, workloads as W

cfgs = W.sweep_configs(n_replicas=512, n=2000)
b = sim.Batch(cfgs, host_threads=os.cpu_count())
b.run()
dev = b.summaries()
t0 = time.time()
dec, eh, wall = Ref().run_batch(cfgs, os.cpu_count() or 1)
same_h = sum(int(d.event_hash == h) for d, h in zip(dev, eh))
same_d = sum(int(d.decisions == x) for d, x in zip(dev, dec))
print(f"replicas {len(cfgs)}: event_hash equal {same_h}, decisions equal {same_d}; "
      f"decisions {sum(dec)}; device kernel {b.kernel_ms():.0f} ms, reference {wall:.1f} s on {os.cpu_count()} threads")
bad = [i for i, (d, h) in enumerate(zip(dev, eh)) if d.event_hash != h]
if bad:
    print("mismatching replicas:", bad[:20])
