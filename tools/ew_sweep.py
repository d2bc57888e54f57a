"""A/B of engine warps per replica CTA (NX_ENGINE_WARPS) on the bench shard."""
import os, sys
sys.path.insert(0, ".")
import bench
from paper_2509_23384_b200 import sim
cfgs = bench.shard_configs(0, 512, 2000)
for ew in sys.argv[1:]:
    os.environ["NX_ENGINE_WARPS"] = ew
    b = sim.Batch(cfgs, host_threads=os.cpu_count())
    b.upload()
    ms = []
    for _ in range(3):
        b.launch(); b.synchronize(); ms.append(b.kernel_ms())
    b.download(); b.synchronize()
    bad = sum(1 for s in b.summaries() if s.status)
    dec = sum(s.decisions for s in b.summaries())
    print(f"engine_warps {ew}: kernel ms {[round(m,1) for m in ms]} -> {dec / (min(ms) / 1e3) / 1e6:.1f} M dec/s, failed {bad}", flush=True)
