"""A/B of launch-time environment settings on the bench shard (same process,
one handle per setting): python tools/env_ab.py "NX_REQ_SMEM=0" "" ..."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench
from paper_2509_23384_b200 import sim
cfgs = bench.shard_configs(0, 512, 2000)
base = dict(os.environ)
for spec in sys.argv[1:] * int(os.environ.get("AB_REPS", "2")):  # each setting AB_REPS times, interleaved
    os.environ.clear(); os.environ.update(base)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    b = sim.Batch(cfgs, host_threads=os.cpu_count())
    b.upload()
    ms = []
    for _ in range(3):
        b.launch(); b.synchronize(); ms.append(b.kernel_ms())
    b.download(); b.synchronize()
    sums = b.summaries()
    bad = sum(1 for s in sums if s.status)
    dec = sum(s.decisions for s in sums)
    h = hash(tuple(s.event_hash for s in sums)) & 0xffff
    print(f"[{spec or 'default'}] kernel ms {[round(m, 1) for m in ms]} -> {dec / (min(ms) / 1e3) / 1e6:.2f} M dec/s "
          f"failed {bad} hashes {h:04x}", flush=True)
    b.close()
