"""Same replica alone vs. 148 copies (one per SM): does full load slow a
replica? SM clocks are sampled during the loaded runs."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench
from paper_2509_23384_b200 import sim, workloads as W
for pol in ("round_robin", "prism"):
    c = W.sweep_replica(10.0, 1, pol, 2000)
    for n in (1, 148):
        b = sim.Batch([c] * n, host_threads=os.cpu_count())
        b.upload()
        with bench.ClockSampler(0) as clk:
            for _ in range(3):
                b.launch(); b.synchronize()
        b.download(); b.synchronize()
        d = [(b.timeline(r)[1] - b.timeline(r)[0]) / 1e6 for r in range(n)]
        print(f"{pol:12s} copies {n:4d}: kernel {b.kernel_ms():7.1f} ms, replica mean {sum(d) / n:7.1f} ms "
              f"max {max(d):7.1f}  clocks {clk.summary()}", flush=True)
        b.close()
