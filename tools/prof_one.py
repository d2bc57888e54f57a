"""One slow sweep replica (10 req/s) alone: the latency-critical case."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_23384_b200 import sim, workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
b = sim.Batch([W.sweep_replica(10.0, 1, "prism", n)])
b.run()
print(f"kernel {b.kernel_ms():.1f} ms, events {b.summaries()[0].events}")
