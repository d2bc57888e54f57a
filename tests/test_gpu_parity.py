"""GPU suite: the sm_100a kernels, called through the C-ABI, against the
reference simulator (oracle/_ref — compiled, unmodified) and the golden
fixtures it produced.

Bit-exact: event_hash (every routing choice, batch composition, token budget
and event time), arrival_hash, every RequestRecord, the TTFT/TPOT/e2e/SLO
metrics and engine shares. Tolerance: the learners' reported p_max (1e-10
on the golden cases with at least 30% bit-identical, 1e-9 at full size
relative; device libm and tree-order accumulation differ from glibc in the
last bits) and K1 predictions (1e-9 fp64, 1e-4 fp32 fast mode).
"""
import json
import math
import tempfile
from pathlib import Path

import numpy as np
import pytest

from cases import static_cases, trace_cases
from oracle_lib import Port, Ref, ref_available

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((ROOT / "tests" / "golden" / "cases.json").read_text())
P_MAX_TOL = 1e-9           # full-size BASELINE configs (test_configs_gpu.py)
GOLDEN_P_MAX_TOL = 1e-10   # the 28 golden cases: largest observed 1.08e-11 (tools/hist_stats.py)


def _checker():
    return Ref() if ref_available() else Port()


def assert_same_summary(want_json: str, got_json: str, tol: float = P_MAX_TOL):
    """Every summary field equal except learners[].p_max (relative `tol`);
    returns (learners whose p_max is bit-identical, learners)."""
    a, b = json.loads(want_json), json.loads(got_json)
    for k in ("seed", "router_policy", "engines", "arrived", "completed", "rejected",
              "unfinished", "arrival_hash", "event_hash", "metrics", "engine_share"):
        assert a[k] == b[k], (k, a[k], b[k])
    assert len(a["learners"]) == len(b["learners"])
    same = 0
    for la, lb in zip(a["learners"], b["learners"]):
        assert la["engine_id"] == lb["engine_id"] and la["samples"] == lb["samples"]
        assert abs(la["p_max"] - lb["p_max"]) <= tol * abs(la["p_max"])
        same += la["p_max"] == lb["p_max"]
    return same, len(a["learners"])


@pytest.fixture(scope="module")
def all_cases(tmp_path_factory):
    from paper_2509_23384_b200 import sim
    td = tmp_path_factory.mktemp("traces")
    c = dict(static_cases())
    c.update(trace_cases(str(td), sim.synth_generate))
    return c


@pytest.fixture(scope="module")
def device_batch(all_cases):
    """Every parity case as ONE device batch (one CTA per replica)."""
    from paper_2509_23384_b200 import sim
    names = sorted(all_cases)
    b = sim.Batch([all_cases[n] for n in names]).run()
    yield names, b
    b.close()


def test_every_case_bit_exact_against_golden(device_batch):
    names, b = device_batch
    sums = b.summaries()
    same = total = 0
    for i, name in enumerate(names):
        want = GOLDEN[name]
        assert sums[i].status == 0, name
        assert f"{sums[i].event_hash:016x}" == want["event_hash"], name
        assert f"{sums[i].arrival_hash:016x}" == want["arrival_hash"], name
        assert sums[i].decisions == want["decisions"], name
        s, t = assert_same_summary(want["summary_json"], b.summary_json(i), GOLDEN_P_MAX_TOL)
        same += s
        total += t
    # drift guard: 70 of the 167 learners' p_max are bit-identical today
    assert same >= 0.3 * total, (same, total)


def test_records_identical_to_reference(device_batch, all_cases):
    names, b = device_batch
    chk = _checker()
    for i, name in enumerate(names):
        want = chk.run(all_cases[name], records=True)
        got = b.records(i)
        assert [r.request_id for r in got] == want["rec_id"], name
        assert [r.engine_id for r in got] == want["rec_engine"], name
        assert [r.first_token_ms for r in got] == want["rec_first"], name
        assert [r.completed_ms for r in got] == want["rec_done"], name
        assert [r.arrival_ms for r in got] == want["rec_arrival"], name


def test_single_replica_equals_batched_replica(all_cases, device_batch):
    """Replicas in one launch are independent: running one alone gives the
    same result as inside the batch."""
    from paper_2509_23384_b200 import sim
    names, b = device_batch
    for name in ("het_prism", "config2_gamma_cv3", "kv_pressure"):
        one = sim.run_simulation(all_cases[name])
        i = names.index(name)
        assert one.event_hash == b.summaries()[i].event_hash
        assert one.summary_json == b.summary_json(i)


def test_rebuild_overlapping_a_launch_keeps_results():
    """nx_sim_rebuild_workloads while the previous launch is in flight (the
    pipelined e2e loop in bench.py): it waits for that launch's H2D copies
    before rewriting the pinned inputs, so both launches give the same
    event hashes, decisions and records as a plain run."""
    from paper_2509_23384_b200 import sim, workloads as W
    cfgs = W.sweep_configs(32, n=300)
    ref = sim.Batch(cfgs).run()
    want = [(x.event_hash, x.decisions) for x in ref.summaries()]
    want_rec = [r.completed_ms for r in ref.records(5)]
    ref.close()
    b = sim.Batch(cfgs)
    for step in range(3):
        b.upload()
        b.launch()
        b.download()
        b.rebuild_workloads(4)  # overlaps the launch
        b.synchronize()
        assert [(x.event_hash, x.decisions) for x in b.summaries()] == want, step
        assert [r.completed_ms for r in b.records(5)] == want_rec, step
    b.close()


def test_sweep_slice_matches_reference_batch():
    from paper_2509_23384_b200 import sim, workloads as W
    cfgs = W.sweep_configs(64, n=300)
    dec, eh, _ = _checker().run_batch(cfgs, 8)
    b = sim.Batch(cfgs).run()
    s = b.summaries()
    assert [x.event_hash for x in s] == eh
    assert [x.decisions for x in s] == dec
    b.close()


def test_sweep_api_rows():
    from paper_2509_23384_b200 import sim, workloads as W
    base = W.config3(n=300)
    res = sim.sweep(base, "rate", [15.0, 30.0, 45.0])
    chk = _checker()
    for row, rate in zip(res["rows"], [15.0, 30.0, 45.0]):
        cfg = json.loads(json.dumps(base))
        cfg["workload"]["rate"] = rate
        want = chk.run(cfg)
        assert row["ok"] and f"{row['result'].event_hash:016x}" == want["event_hash"]


def test_host_errors_raise_reference_classes():
    from paper_2509_23384_b200 import sim, workloads as W
    cfg = W.config1(n=200)
    cfg["engines"][0].update(scheduler_policy="prefill_priority", m_max=128, q_max=64)
    cfg["scheduler"] = {"q_max": 64}
    with pytest.raises(RuntimeError):
        sim.run_simulation(cfg)
    with pytest.raises(RuntimeError):
        sim.run_simulation({"engines": []})


# ---- K1 perf-model evaluator ----------------------------------------------------
def _rows():
    from paper_2509_23384_b200 import perf_model as pm
    return [pm.PROFILES["fast"], pm.PROFILES["medium"], pm.PROFILES["slow"], pm.DEFAULT_PRIORS,
            pm.PerfParams(1.5, 2.0, 1.2, 0.3, 0.01, 8.0, 0.7, 0.05)]


def test_k1_known_answers():
    from paper_2509_23384_b200 import perf_model as pm
    p = pm.PerfParams(p_max=10.0, kB=0.5, kS=0.01)
    assert pm.throughput(p, (2, 100)) == pytest.approx(3.995764008937280535437497, rel=1e-13)
    q = pm.PerfParams(1.5, 2.0, 1.2, 0.3, 0.01, 8.0, 0.7, 0.05)
    assert pm.predict_latency(q, (1, 1)) == pytest.approx(18.10206826697007059858764, rel=1e-13)
    sat = pm.PerfParams(tau0=5.0, kB=1000.0, kS=1000.0)
    assert pm.predict_latency(sat, (4, 100)) == pytest.approx(105.0, rel=1e-8)
    assert pm.throughput(pm.PerfParams(p_max=17.0, kB=1000.0, kS=1000.0), (1000000, 1000000000)) < 17.0


@pytest.mark.parametrize("mode,tol", [(0, 1e-9), (1, 1e-4)])
def test_k1_random_records_against_oracle(mode, tol):
    from paper_2509_23384_b200 import perf_model as pm
    rows = _rows()
    rng = np.random.default_rng(11)
    n = 1_000_003  # odd: exercises the vector tail
    idx = rng.integers(0, len(rows), n)
    b = rng.integers(1, 1024, n)
    s = b + rng.integers(0, 200_000, n)
    T, thr = pm.eval_host(rows, idx, b, s, mode=mode)
    port = Port()
    worst = 0.0
    for k, r in enumerate(rows):
        m = idx == k
        Tr, thr_r = port.perf_eval(pm._row(r), b[m], s[m])
        worst = max(worst, float(np.max(np.abs(T[m] - Tr) / Tr)),
                    float(np.max(np.abs(thr[m] - thr_r) / thr_r)))
        if mode == 0 and k == 0:  # the fast profile evaluates bit-identically
            assert np.array_equal(T[m], Tr)
    assert worst <= tol


def test_k1_monotone_bisection_predicate_bitwise():
    """The LENS bisection predicate T(b, S) <= target must agree bit for bit:
    reproduce test_lens.cpp:136-152's vectors (200 random targets)."""
    from paper_2509_23384_b200 import perf_model as pm
    rng = np.random.default_rng(29)
    for i in range(50):
        p = pm.PROFILES["fast" if i % 2 else "medium"]
        p = pm.PerfParams(rng.uniform() * 10.0, p.w0, p.ws, rng.uniform(), p.tauS, p.p_max, p.kB,
                          0.01 + rng.uniform() * 0.2)
        b = int(rng.integers(1, 33))
        s = np.arange(b, 4097)
        T, _ = pm.eval_host([p], np.zeros(len(s)), np.full(len(s), b), s, want_thr=False)
        Tr, _ = Port().perf_eval(pm._row(p), np.full(len(s), b), s)
        target = Tr[0] * (0.5 + rng.uniform() * 4.0)
        assert np.array_equal(T <= target, Tr <= target)


def test_k1_rejects_invalid_like_reference():
    from paper_2509_23384_b200 import perf_model as pm
    with pytest.raises(ValueError):
        pm.predict_latency(pm.PerfParams(), (0, 5))
    with pytest.raises(ValueError):
        pm.predict_latency(pm.PerfParams(), (4, 3))
    with pytest.raises(ValueError):
        pm.predict_latency(pm.PerfParams(p_max=-1.0), (1, 1))


def test_smoke_entry_point():
    import sys
    sys.path.insert(0, str(ROOT))
    import __graft_entry__
    __graft_entry__.smoke()


def test_exclusive_sm_schedule_gives_identical_results(all_cases, monkeypatch):
    """The kernel's replica scheduling (exclusive SMs for the longest
    replicas, then the shared queue) changes only where replicas run."""
    from paper_2509_23384_b200 import sim
    names = sorted(all_cases)
    monkeypatch.setenv("NX_EXCL_SMS", "6")
    b = sim.Batch([all_cases[n] for n in names]).run()
    try:
        sums = b.summaries()
        for i, name in enumerate(names):
            assert f"{sums[i].event_hash:016x}" == GOLDEN[name]["event_hash"], name
            assert sums[i].decisions == GOLDEN[name]["decisions"], name
    finally:
        b.close()
