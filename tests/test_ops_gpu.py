"""GPU suite for the batched operators (K2 nx_lens_schedule, K3
nx_prism_route, K4 nx_refit), called through the C-ABI, against the
reference's own operators: golden fixtures made by oracle/_ref
(tests/golden/make_ops_golden.py) and, where the compiled reference is
present, live calls on the same inputs.

Bit-exact: every plan's (b, s, overload), every allocation, every routing
choice and degraded flag, the echoed report view, every learner's
updated flag and counters, every error status. Tolerance: floating values
computed through device libm (predicted/target latency 1e-12 relative,
route scores/factors 1e-12, refit params 1e-9 — the simulator's p_max
bound).
"""
import json
from pathlib import Path

import numpy as np
import pytest

import ops_cases
from paper_2509_23384_b200 import abi, learner, lens, router

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "ops_golden.json").read_text())


def _close(a, b, tol):
    a, b = float(a), float(b)
    return a == b or abs(a - b) <= tol * max(abs(a), abs(b))


def _unhex(v):
    return float.fromhex(v)


# ---- schedule_baseline (engine.cpp:61-108) ------------------------------------------
def test_baseline_batch_matches_reference_schedule_baseline():
    cases = ops_cases.baseline_cases()
    probs = np.zeros(len(cases), dtype=abi.BASELINE_PROBLEM)
    rem, off = [], 0
    for i, c in enumerate(cases):
        r = [p - f for p, f in zip(c["prompt"], c["prefilled"])]
        probs[i] = lens.baseline_record(c["policy"], c["n_run"], len(r), off, c["params"], c["m_max"],
                                        c["q_max"], c["static_budget"], c["engine_id"])
        rem += r
        off += len(r)
    out, tok = lens.schedule_baseline_batch(probs, np.asarray(rem, dtype=np.int32), raise_errors=False)
    for i, want in enumerate(GOLD["baseline"]):
        p = out[i]
        assert int(p["status"]) == want["status"], i
        if want["status"]:
            continue
        assert (int(p["b"]), int(p["s"])) == (want["b"], want["s"]), i
        assert _close(p["predicted_ms"], _unhex(want["predicted"]), 1e-12), i
        w0 = int(probs[i]["wait_off"])
        alloc = [[j, 1, 0] for j in range(int(p["n_decode"]))]
        alloc += [[1000 + k, int(tok[w0 + k]), 1] for k in range(int(p["n_prefill"]))]
        assert alloc == want["alloc"], i


def test_baseline_scalar_api_mirrors_reference():
    runs = [lens.Request(id=100 + i, prompt_len=64, prefilled=64) for i in range(5)]
    waits = [lens.Request(id=p, prompt_len=p) for p in (300, 400)]
    plan = lens.schedule_baseline(lens.PREFILL_PRIORITY, waits, runs, ops_cases.FAST, q_max=64)
    assert (plan.b, plan.s) == (2, 700) and all(a.is_prefill for a in plan.allocations)
    plan = lens.schedule_baseline(lens.PREFILL_PRIORITY, [], runs, ops_cases.FAST, q_max=64)
    assert (plan.b, plan.s) == (5, 5)
    with pytest.raises(RuntimeError):
        lens.schedule_baseline(lens.PREFILL_PRIORITY, [lens.Request(id=1, prompt_len=9000)], [],
                               ops_cases.FAST)
    with pytest.raises(ValueError):
        lens.schedule_baseline(lens.STATIC_CHUNKED, [], runs, ops_cases.FAST, q_max=4, m_max=8192)


# ---- K2 --------------------------------------------------------------------------
@pytest.fixture(scope="module")
def lens_run():
    cases = ops_cases.lens_cases()
    probs = np.zeros(len(cases), dtype=abi.LENS_PROBLEM)
    rem, off = [], 0
    for i, c in enumerate(cases):
        r = [p - f for p, f in zip(c["prompt"], c["prefilled"])]
        probs[i] = lens.problem_record(
            c["n_run"], len(r), off, lens.SLOSpec(c["ttft"], c["tpot"]),
            lens.TradeoffModel(*c["tm"]), c["params"],
            lens.SchedulerConfig(c["m_max"], c["q_max"], c["n_iters"], c["eps"], c["q_ref"]))
        rem += r
        off += len(r)
    plans, alloc = lens.schedule_batch(probs, np.asarray(rem, dtype=np.int32), raise_errors=False)
    return cases, probs, plans, alloc


def test_lens_batch_matches_reference_schedule_step(lens_run):
    cases, probs, plans, alloc = lens_run
    assert len(GOLD["lens"]) == len(cases)
    exact_pred = 0
    for i, (c, want) in enumerate(zip(cases, GOLD["lens"])):
        p = plans[i]
        assert int(p["status"]) == want["status"], i
        if want["status"]:
            continue
        assert (int(p["b"]), int(p["s"]), int(p["overload"])) == (want["b"], want["s"], want["overload"]), i
        assert _close(p["predicted_ms"], _unhex(want["predicted"]), 1e-12), i
        assert _close(p["target_ms"], _unhex(want["target"]), 1e-12), i
        exact_pred += float(p["predicted_ms"]) == _unhex(want["predicted"])
        got = [(k, 1, 0) for k in range(int(p["n_decode"]))]
        off = int(probs[i]["wait_off"])
        got += [(1000 + k, int(alloc[off + k]), 1) for k in range(int(p["n_prefill"]))]
        assert got == [tuple(a) for a in want["alloc"]], i
    assert exact_pred >= 0.95 * sum(w["status"] == 0 for w in GOLD["lens"])


def test_lens_plans_respect_feasibility_invariants(lens_run):
    # tests/test_lens.cpp:332-372 on every valid device plan
    cases, probs, plans, alloc = lens_run
    for i, c in enumerate(cases):
        p = plans[i]
        if p["status"] or (c["n_run"] == 0 and not c["prompt"]):
            continue
        assert p["b"] <= c["q_max"] and p["s"] <= c["m_max"]
        assert p["b"] == p["n_decode"] + p["n_prefill"]
        off = int(probs[i]["wait_off"])
        toks = [int(alloc[off + k]) for k in range(int(p["n_prefill"]))]
        rem = [pp - f for pp, f in zip(c["prompt"], c["prefilled"])]
        assert all(1 <= t <= r for t, r in zip(toks, rem))
        assert int(p["n_decode"]) + sum(toks) == p["s"]
        if not p["overload"]:
            assert p["n_decode"] == c["n_run"]


def test_lens_fast_fp32_mode(lens_run):
    """NX_FAST_FP32 (include/nx_sched.h): same validation and statuses, every
    plan feasible, predicted_ms within 1e-4 of the fp64 model for the plan
    it chose, and the same (b, s) as the deterministic mode on nearly every
    decision (they may differ only where float rounding reorders two
    candidates or a probe and the target; SURVEY App. A.5 validates the fast
    mode statistically)."""
    cases, probs, plans64, _ = lens_run
    rem = []
    for c in cases:
        rem += [p - f for p, f in zip(c["prompt"], c["prefilled"])]
    rem = np.asarray(rem, dtype=np.int32)
    plans, alloc = lens.schedule_batch(probs, rem, raise_errors=False, mode=lens.NX_FAST_FP32)
    same = valid = 0
    for i, c in enumerate(cases):
        p, q = plans[i], plans64[i]
        assert int(p["status"]) == int(q["status"]), i
        if p["status"] or (c["n_run"] == 0 and not c["prompt"]):
            continue
        valid += 1
        assert p["b"] <= c["q_max"] and p["s"] <= c["m_max"]
        assert p["b"] == p["n_decode"] + p["n_prefill"]
        off = int(probs[i]["wait_off"])
        toks = [int(alloc[off + k]) for k in range(int(p["n_prefill"]))]
        assert all(1 <= t <= r for t, r in zip(toks, rem[off:off + len(toks)]))
        assert int(p["n_decode"]) + sum(toks) == p["s"]
        assert _close(p["target_ms"], q["target_ms"], 0.0)  # target stays fp64
        want = ops_cases._predict(list(probs[i]["params"]), int(p["b"]), int(p["s"]))
        assert _close(p["predicted_ms"], want, 1e-4), (i, float(p["predicted_ms"]), want)
        same += (int(p["b"]), int(p["s"])) == (int(q["b"]), int(q["s"]))
    assert valid > 400 and same >= 0.95 * valid, (same, valid)
    with pytest.raises(ValueError):
        lens.schedule_batch(probs[:1], rem, mode=7)


def test_lens_scalar_api_mirrors_reference():
    R = [lens.Request(id=i, prompt_len=64, prefilled=64) for i in range(4)]
    W = [lens.Request(id=10 + i, prompt_len=p) for i, p in enumerate([100, 300, 5, 2000])]
    plan = lens.schedule_step(W, R, lens.SLOSpec(40.0, 12.0), lens.TradeoffModel(100.0, 10.0, 200.0, 1.0),
                              ops_cases.MEDIUM, lens.SchedulerConfig())
    assert plan.b == len(plan.allocations) and plan.s == sum(a.tokens for a in plan.allocations)
    assert [a.request_id for a in plan.allocations[:4]] == [0, 1, 2, 3]
    with pytest.raises(ValueError):
        lens.schedule_step(W, R, lens.SLOSpec(40.0, -1.0), lens.TradeoffModel(), ops_cases.FAST,
                           lens.SchedulerConfig())


# ---- K3 --------------------------------------------------------------------------
def _route_inputs(cases):
    groups = np.zeros(len(cases), dtype=abi.ROUTE_GROUP)
    reps, reqs, smaps = [], [], []
    eo = ro = so = 0
    for g, c in enumerate(cases):
        G = groups[g]
        cfg = c["cfg9"]
        G["weights"] = cfg[:4]
        (G["beta_aff"], G["latency_knee"], G["latency_scale_ms"], G["load_half_ms"],
         G["capacity_headroom"]) = cfg[4:9]
        G["staleness_limit_ms"] = 1000.0
        G["ttft_slo_ms"] = c["ttft"]
        G["rng"] = router.router_rng_state(c["seed"])
        G["policy"], G["n_engines"] = c["policy"], len(c["ids"])
        n = len(c["ids"])
        rows = np.zeros(n, dtype=abi.ENGINE_REPORT)
        for e in range(n):
            (rows[e]["l_hat_ms"], rows[e]["w_load_tokens"], rows[e]["m_free_tokens"],
             rows[e]["p_max"], rows[e]["reported_at_ms"]) = c["states5"][e]
            rows[e]["queue_len"], rows[e]["engine_id"] = c["qlen"][e], c["ids"][e]
            rows[e]["has_report"], rows[e]["static_weight"] = c["has_report"][e], c["static_w"][e]
        # Router::on_completion replay: decode-length EMA + session memory (router.cpp:83-92)
        lbar = 128.0
        sm = np.full(c["n_sessions"], -1, dtype=np.int32)
        for eng, ses, dec in zip(c["comp_engine"], c["comp_session"], c["comp_decode"]):
            if eng not in c["ids"]:
                continue
            lbar = lbar + 0.05 * (float(dec) - lbar)
            if lbar < 1.0:
                lbar = 1.0
            sm[ses] = c["ids"].index(eng)
        G["l_bar_ema"] = lbar
        q = np.zeros(len(c["req_prompt"]), dtype=abi.ROUTE_REQUEST)
        q["now_ms"], q["prompt_len"], q["session"] = c["req_now"], c["req_prompt"], c["req_session"]
        G["engine_off"], G["request_off"], G["session_off"] = eo, ro, so
        G["n_requests"], G["n_sessions"] = q.size, sm.size
        eo += n
        ro += q.size
        so += sm.size
        reps.append(rows)
        reqs.append(q)
        smaps.append(sm)
    return groups, np.concatenate(reps), np.concatenate(reqs), np.concatenate(smaps)


def test_route_batch_matches_reference_router():
    cases = ops_cases.route_cases()
    groups, reps, reqs, smap = _route_inputs(cases)
    dec, st = router.route_batch(groups, reps, reqs, smap, raise_errors=False)
    for g, (c, want) in enumerate(zip(cases, GOLD["route"])):
        assert int(st[g]) == want["status"], g
        if want["status"]:
            continue
        o = int(groups[g]["request_off"])
        m = len(c["req_prompt"])
        assert dec["engine_id"][o:o + m].tolist() == want["engine"], g
        assert dec["degraded"][o:o + m].tolist() == want["degraded"], g
        for k in range(m):
            assert _close(dec["score"][o + k], _unhex(want["score"][k]), 1e-12), (g, k)
            for j in range(4):
                assert _close(dec["factors"][o + k][j], _unhex(want["factors"][k][j]), 1e-12), (g, k, j)
        eo = int(groups[g]["engine_off"])
        n = len(c["ids"])
        for e in range(n):  # the Router's report view after the dispatch echoes
            if not c["has_report"][e]:
                continue
            assert int(reps["queue_len"][eo + e]) == want["qlen"][e], (g, e)
            assert float(reps["w_load_tokens"][eo + e]) == _unhex(want["states5"][e][1]), (g, e)


def test_route_fast_fp32_mode():
    """NX_FAST_FP32 for K3: same statuses, and the deterministic mode's
    choices on nearly every routing decision (they may differ only where two
    engines' float scores tie or swap within rounding; a group's later routes
    then see a different dispatch echo, so they are compared only up to its
    first difference). Scores and factors within 1e-4 relative there (the
    fast mode's bound; the stale-report blend 1 + (f - 1) b cancels when b is
    near 1, which turns float rounding into ~1e-5)."""
    cases = ops_cases.route_cases()
    groups, reps, reqs, smap = _route_inputs(cases)
    d64, s64 = router.route_batch(groups, reps, reqs, smap, raise_errors=False)
    groups, reps, reqs, smap = _route_inputs(cases)
    d32, s32 = router.route_batch(groups, reps, reqs, smap, raise_errors=False, mode=1)
    assert (s32 == s64).all()
    agree = total = groups_ok = n_groups = 0
    for g, c in enumerate(cases):
        if s64[g]:
            continue
        n_groups += 1
        o, m = int(groups[g]["request_off"]), len(c["req_prompt"])
        total += m
        for k in range(o, o + m):
            if d32["engine_id"][k] != d64["engine_id"][k]:
                break
            agree += 1
            assert _close(d32["score"][k], d64["score"][k], 1e-4), (g, k)
            for j in range(4):
                assert _close(d32["factors"][k][j], d64["factors"][k][j], 1e-4), (g, k, j)
        else:
            groups_ok += 1
    assert total > 1000 and agree >= 0.9 * total and groups_ok >= 0.9 * n_groups, (agree, total, groups_ok, n_groups)
    with pytest.raises(ValueError):
        router.route_batch(*_route_inputs(cases[:1]), mode=3)


def test_route_errors_match_reference():
    c = ops_cases.route_cases()[0]
    groups, reps, reqs, smap = _route_inputs([c])
    groups["n_engines"] = 0  # Router::route with no engines: std::runtime_error
    with pytest.raises(RuntimeError):
        router.route_batch(groups, reps, reqs, smap)
    groups, reps, reqs, smap = _route_inputs([c])
    groups["beta_aff"] = 0.5  # invalid RouterConfig: std::invalid_argument
    with pytest.raises(ValueError):
        router.route_batch(groups, reps, reqs, smap)


# ---- K4 --------------------------------------------------------------------------
def test_refit_batch_matches_reference_learner():
    metas, b, s, y = ops_cases.refit_cases()
    res = {}
    for kind in (learner.LINEAR, learner.STRUCTURAL):
        idx = [i for i, m in enumerate(metas) if m["kind"] == kind]
        probs = np.zeros(len(idx), dtype=abi.REFIT_PROBLEM)
        for j, i in enumerate(idx):
            m = metas[i]
            probs[j] = learner.problem_record(
                m["priors"], learner.LearnerConfig(m["long_w"], m["short_w"], 1 << 30, (1 << 30) - 1,
                                                   m["min_s"]), m["off"], m["n"])
        out = learner.refit_batch(kind, probs, b, s, y, raise_errors=False)
        for j, i in enumerate(idx):
            res[i] = out[j]
    for i, want in enumerate(GOLD["refit"]):
        r = res[i]
        assert int(r["status"]) == want["status"], i
        if want["status"]:
            continue
        assert int(r["updated"]) == want["updated"], i
        assert r["counters"].tolist() == want["counters"], i
        for k in range(8):
            assert _close(r["params"][k], _unhex(want["params"][k]), 1e-9), (i, k)
