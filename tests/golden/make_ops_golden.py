"""Regenerates tests/golden/ops_golden.json from the UNMODIFIED reference
operators (oracle/_ref/libservesim_ref.so: servesim::schedule_step,
Router::route, OnlineLearner::update_linear / update_structural called by
oracle/ref_driver.cpp). Run here (where /root/reference exists):

    python tests/golden/make_ops_golden.py

Cases come from tests/ops_cases.py (seeded); the file pins a digest of the
generated inputs so a test on another machine can prove it regenerated the
same cases before comparing.
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import ops_cases  # noqa: E402
from oracle_lib import Ref  # noqa: E402
from paper_2509_23384_b200 import router as R  # noqa: E402


def digest(obj) -> str:
    h = hashlib.sha256()
    if isinstance(obj, tuple):
        for a in obj:
            h.update(json.dumps(a, sort_keys=True).encode() if not isinstance(a, np.ndarray) else a.tobytes())
    else:
        h.update(json.dumps(obj, sort_keys=True).encode())
    return h.hexdigest()


def hx(v) -> str:
    return float(v).hex()


def main():
    ref = Ref()
    lens = ops_cases.lens_cases()
    lens_out = []
    for c in lens:
        r = ref.schedule_step(c["n_run"], c["prompt"], c["prefilled"], c["ttft"], c["tpot"], c["tm"],
                              c["params"], c["m_max"], c["q_max"], c["n_iters"], c["eps"], c["q_ref"])
        if r["status"] == 0:
            r["predicted"], r["target"] = hx(r["predicted"]), hx(r["target"])
        lens_out.append(r)
    routes = ops_cases.route_cases()
    route_out = []
    for c in routes:
        r = ref.route_group(c["policy"], c["cfg9"], c["ttft"], c["tpot"], c["seed"], c["ids"],
                            c["static_w"], c["states5"], c["qlen"], c["has_report"], c["comp_engine"],
                            c["comp_session"], c["comp_decode"], c["req_prompt"], c["req_session"],
                            c["req_now"])
        if r["status"] == 0:
            r = {"status": 0, "engine": r["engine"].tolist(), "score": [hx(x) for x in r["score"]],
                 "factors": [[hx(x) for x in row] for row in r["factors"]],
                 "degraded": r["degraded"].tolist(),
                 "states5": [[hx(x) for x in row] for row in r["states5"]], "qlen": r["qlen"].tolist()}
        route_out.append(r)
    metas, b, s, y = ops_cases.refit_cases()
    refit_out = []
    for m in metas:
        sl = slice(m["off"], m["off"] + m["n"])
        r = ref.learner_refit(m["kind"], m["priors"], m["long_w"], m["short_w"], m["min_s"],
                              b[sl], s[sl], y[sl])
        if r["status"] == 0:
            r = {"status": 0, "params": [hx(x) for x in r["params"]], "updated": r["updated"],
                 "counters": r["counters"].tolist()}
        refit_out.append(r)
    base = ops_cases.baseline_cases()
    base_out = []
    for c in base:
        r = ref.schedule_baseline(c["policy"], c["n_run"], c["prompt"], c["prefilled"], c["params"],
                                  c["m_max"], c["q_max"], c["static_budget"], c["engine_id"])
        if r["status"] == 0:
            r["predicted"] = hx(r["predicted"])
        base_out.append(r)
    out = {
        "digest": {"lens": digest(lens), "route": digest(routes),
                   "refit": digest((metas, b, s, y)), "baseline": digest(base)},
        "lens": lens_out, "route": route_out, "refit": refit_out, "baseline": base_out,
    }
    (ROOT / "tests" / "golden" / "ops_golden.json").write_text(json.dumps(out))
    bad = sum(r["status"] != 0 for r in lens_out + route_out + refit_out + base_out)
    print(f"lens {len(lens_out)} route {len(route_out)} refit {len(refit_out)} "
          f"baseline {len(base_out)} (error cases {bad})")


if __name__ == "__main__":
    main()
