import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2509_23384_b200 import sim, workloads as W
n = int(sys.argv[1])
c = W.sweep_replica(10.0, 1, "round_robin", 2000)
b = sim.Batch([c] * n); b.run(); print("kernel", b.kernel_ms())
