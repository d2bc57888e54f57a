"""Device time of single BASELINE-config replicas (kernel ms of one launch
each, best of `reps`): python tools/config_time.py [reps]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2509_23384_b200 import sim, workloads as W
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for name, cfg in (("config3_100k", W.config3(n=100000)), ("config1_1k", W.config1(n=1000))):
    b = sim.Batch([cfg])
    b.upload()
    ms = []
    for _ in range(reps):
        b.launch(); b.synchronize(); ms.append(b.kernel_ms())
    b.download(); b.synchronize()
    s = b.summaries()[0]
    print(f"{name}: kernel ms {[round(m, 1) for m in ms]} decisions {s.decisions} hash {s.event_hash:016x}", flush=True)
    b.close()
