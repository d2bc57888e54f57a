"""Ad-hoc device-vs-reference comparison (run under gpurun)."""
import json, sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from oracle_lib import Ref
from paper_2509_23384_b200 import workloads as W, sim
ref = Ref()
cases = [W.config1(n=50), W.config1(n=200), W.config1(seed=2, rate=4, n=300), W.config3(n=2000),
         W.config3(n=1500, policy="round_robin"), W.config3(n=1500, policy="least_loaded"),
         W.config3(n=1500, policy="latency_based"), W.config3(n=1500, policy="weighted"),
         W.config3(n=1500, policy="session_affinity")]
ok = 0
for c in cases:
    a = ref.run(c, True)
    t = time.time()
    try:
        b = sim.run_simulation(c)
    except Exception as e:
        print("DEVICE ERROR", c["router"]["policy"], c["workload"]["n"], repr(e)); continue
    dt = time.time() - t
    same = a["event_hash"] == f"{b.event_hash:016x}"
    ssame = a["summary_json"] == b.summary_json
    ok += same and ssame
    print(c["router"]["policy"], c["workload"]["n"], a["event_hash"], f"{b.event_hash:016x}", "HASH_OK" if same else "HASH_DIFF",
          "SUM_OK" if ssame else "SUM_DIFF", a["decisions"], b.decisions, b.events, f"{dt:.2f}s")
    if not ssame:
        print(a["summary_json"]); print(b.summary_json)
print(f"{ok}/{len(cases)} identical")
