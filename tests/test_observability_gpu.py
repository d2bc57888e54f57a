"""Observability outputs written from device buffers,
against the reference simulator on the same config: output.dir files
(summary.json, requests.csv, plans.jsonl, routing.jsonl — sim.cpp:393-413)
and RunResult::learner_history (sim.cpp:322-327).

Exact: every integer field, every row count and order, summary.json and
requests.csv bytes (p_max in summary.json within 1e-10 like the golden
parity suite). Tolerance: device-libm floats in the logs — predicted
latencies 1e-12 relative; route factors (which read the reported learner
p_max) 1e-11; every learner coefficient of every history snapshot 1e-9, with
at least a quarter of them bit-identical.
"""
import copy
import json
from pathlib import Path

import pytest

from cases import static_cases
from oracle_lib import Ref, ref_available
from paper_2509_23384_b200 import sim

pytestmark = pytest.mark.gpu

CASES = ["c1_small", "het_prism", "het_weighted", "prefill_priority", "mixed_policies"]


def _close(a, b, tol):
    return a == b or abs(a - b) <= tol * max(abs(a), abs(b))


def _rows(path: Path):
    return [json.loads(x) for x in path.read_text().splitlines()]


def _cmp_rows(want, got, exact, tol):
    assert len(want) == len(got)
    for w, g in zip(want, got):
        assert list(w) == list(g)  # same keys, same order
        for k in w:
            if k in exact:
                assert w[k] == g[k], (k, w, g)
            else:
                assert _close(float(w[k]), float(g[k]), tol), (k, w, g)


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
@pytest.mark.parametrize("name", CASES)
def test_output_files_and_history_match_reference(name, tmp_path):
    base = copy.deepcopy(static_cases()[name])
    base["workload"]["n"] = min(base["workload"].get("n", 200), 200)
    base["record_learner_history"] = True
    out = {}
    for who in ("ref", "dev"):
        cfg = copy.deepcopy(base)
        cfg["output"] = {"dir": str(tmp_path / who), "plans_jsonl": "plans.jsonl",
                         "routing_jsonl": "routing.jsonl"}
        out[who] = cfg
    want = Ref().run(out["ref"], records=True)
    got = sim.run_simulation(out["dev"])
    R, D = tmp_path / "ref", tmp_path / "dev"
    assert (R / "requests.csv").read_bytes() == (D / "requests.csv").read_bytes()
    a, b = json.loads((R / "summary.json").read_text()), json.loads((D / "summary.json").read_text())
    for la, lb in zip(a.pop("learners"), b.pop("learners")):
        assert la["engine_id"] == lb["engine_id"] and la["samples"] == lb["samples"]
        assert _close(la["p_max"], lb["p_max"], 1e-10)
    assert a == b
    _cmp_rows(_rows(R / "plans.jsonl"), _rows(D / "plans.jsonl"),
              {"engine_id", "b", "s", "sim_time"}, 1e-12)
    # route factors read the engines' reported p_max (largest observed
    # difference 2e-13, tools/hist_stats.py)
    _cmp_rows(_rows(R / "routing.jsonl"), _rows(D / "routing.jsonl"),
              {"request_id", "chosen_engine", "sim_time"}, 1e-11)
    hist = want["learner_history"]
    assert len(hist) == len(got.learner_history) > 0
    same = total = 0
    for (e0, t0, n0, p0), (e1, t1, n1, p1) in zip(hist, got.learner_history):
        assert (e0, t0, n0) == (e1, t1, n1)
        # every coefficient of every snapshot, not just the summary's p_max:
        # w0 = a / c out of the ridge-anchored 5x5 solve amplifies the device
        # libm ulps in the noise and f_B / f_S values (largest observed on
        # these cases 1.07e-10, prefill_priority; tools/hist_stats.py), so 1e-9
        bad = [(i, x, y) for i, (x, y) in enumerate(zip(p0, p1)) if not _close(x, y, 1e-9)]
        assert not bad, (e0, t0, n0, bad)
        same += sum(x == y for x, y in zip(p0, p1))
        total += len(p0)
    # drift guard: a third to over half of all coefficients are bit-identical
    # to the reference's (observed 33-58% per case); a systematic drift that
    # stayed inside the tolerance would show up here first
    assert same >= 0.25 * total, (same, total)
