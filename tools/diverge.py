"""First divergence between the device and the compiled reference for one
golden case: learner-history snapshots (engine, time, samples, params) and
plan log rows. Usage: diverge.py <case name>"""
import copy, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from cases import static_cases
from oracle_lib import Ref
from paper_2509_23384_b200 import sim

name = sys.argv[1]
cfg = copy.deepcopy(static_cases()[name])
cfg["record_learner_history"] = True
want = Ref().run(copy.deepcopy(cfg), records=True)
got = sim.run_simulation(copy.deepcopy(cfg))
H0, H1 = want["learner_history"], got.learner_history
print(f"snapshots ref {len(H0)} dev {len(H1)}")
worst = 0.0
for k, ((e0, t0, n0, p0), (e1, t1, n1, p1)) in enumerate(zip(H0, H1)):
    rel = max(abs(x - y) / max(abs(x), abs(y), 1e-300) for x, y in zip(p0, p1))
    worst = max(worst, rel)
    if (e0, t0, n0) != (e1, t1, n1) or rel > 1e-6:
        print(f"first divergence at snapshot {k}: ref {(e0, t0, n0)} dev {(e1, t1, n1)} rel {rel:.3e}")
        print("  ref params", p0)
        print("  dev params", p1)
        if k:
            print("  previous ref", H0[k - 1])
            print("  previous dev", H1[k - 1])
        break
    if rel > 1e-10:
        print(f"snapshot {k} {(e0, t0, n0)} rel {rel:.3e}")
print(f"max rel before divergence {worst:.3e}")
