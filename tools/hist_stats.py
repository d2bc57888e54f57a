import copy, json, sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from cases import static_cases
from oracle_lib import Ref
from paper_2509_23384_b200 import sim
import numpy as np
for name in ["c1_small", "het_prism", "het_weighted", "prefill_priority", "mixed_policies"]:
    base = copy.deepcopy(static_cases()[name])
    base["workload"]["n"] = min(base["workload"].get("n", 200), 200)
    base["record_learner_history"] = True
    want = Ref().run(copy.deepcopy(base), records=True)
    got = sim.run_simulation(copy.deepcopy(base))
    same = tot = 0; worst = 0.0; snaps_exact = 0
    for (e0, t0, n0, p0), (e1, t1, n1, p1) in zip(want["learner_history"], got.learner_history):
        ex = True
        for x, y in zip(p0, p1):
            tot += 1
            if x == y: same += 1
            else:
                ex = False
                worst = max(worst, abs(x - y) / max(abs(x), abs(y)))
        snaps_exact += ex
    print(name, "snapshots", len(want["learner_history"]), "bit-identical snapshots", snaps_exact, "coeffs identical", same, "/", tot, "worst rel", worst)
    sw = want.get("summary") or {}

# summary p_max over the golden cases, and route factors / p_max of the
# observability cases (written output files)
import tempfile
from pathlib import Path
from cases import trace_cases
GOLDEN = json.loads(Path("tests/golden/cases.json").read_text())
td = tempfile.mkdtemp()
allc = dict(static_cases()); allc.update(trace_cases(td, sim.synth_generate))
names = sorted(allc)
b = sim.Batch([allc[n] for n in names]).run()
worst = 0.0; same = tot = 0
for i, n in enumerate(names):
    a = json.loads(GOLDEN[n]["summary_json"]); d = json.loads(b.summary_json(i))
    for la, lb in zip(a["learners"], d["learners"]):
        tot += 1; same += la["p_max"] == lb["p_max"]
        if la["p_max"] != lb["p_max"]:
            worst = max(worst, abs(la["p_max"] - lb["p_max"]) / abs(la["p_max"]))
print("golden summaries: learners", tot, "p_max identical", same, "worst rel", worst)
b.close()
for name in ["c1_small", "het_prism", "het_weighted", "prefill_priority", "mixed_policies"]:
    base = copy.deepcopy(static_cases()[name]); base["workload"]["n"] = min(base["workload"].get("n", 200), 200)
    out = {}
    for who in ("ref", "dev"):
        cfg = copy.deepcopy(base)
        cfg["output"] = {"dir": f"{td}/{name}_{who}", "plans_jsonl": "plans.jsonl", "routing_jsonl": "routing.jsonl"}
        out[who] = cfg
    Ref().run(out["ref"], records=True); sim.run_simulation(out["dev"])
    R = [json.loads(x) for x in Path(f"{td}/{name}_ref/routing.jsonl").read_text().splitlines()]
    D = [json.loads(x) for x in Path(f"{td}/{name}_dev/routing.jsonl").read_text().splitlines()]
    w = 0.0; s = t = 0
    for r, d in zip(R, D):
        for k in r:
            if k in ("request_id", "chosen_engine", "sim_time"): continue
            x, y = float(r[k]), float(d[k]); t += 1; s += x == y
            if x != y: w = max(w, abs(x - y) / max(abs(x), abs(y)))
    P = [json.loads(x) for x in Path(f"{td}/{name}_ref/plans.jsonl").read_text().splitlines()]
    Q = [json.loads(x) for x in Path(f"{td}/{name}_dev/plans.jsonl").read_text().splitlines()]
    wp = 0.0; sp = tp = 0
    for r, d in zip(P, Q):
        for k in r:
            if k in ("engine_id", "b", "s", "sim_time"): continue
            x, y = float(r[k]), float(d[k]); tp += 1; sp += x == y
            if x != y: wp = max(wp, abs(x - y) / max(abs(x), abs(y)))
    print(name, "routing floats identical", s, "/", t, "worst rel", w, "| plan floats identical", sp, "/", tp, "worst rel", wp)
