"""Run the bench shard once and print the failing replicas' error slots."""
import sys, collections
sys.path.insert(0, ".")
import bench
from paper_2509_23384_b200 import sim
cfgs = bench.shard_configs(0, int(sys.argv[1]) if len(sys.argv) > 1 else 512, 2000)
b = sim.Batch(cfgs).run()
sums = b.summaries()
bad = [i for i, s in enumerate(sums) if s.status != 0]
print("failed", len(bad), "of", len(sums))
cnt = collections.Counter((sums[i].status, b.error(i)) for i in bad)
print(cnt.most_common(10))
for i in bad[:5]:
    s = sums[i]
    print(i, cfgs[i]["router"], cfgs[i]["workload"].get("rate_per_s"), s.status, b.error(i), s.arrived, s.events)
