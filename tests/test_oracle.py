"""CPU suite: pins the oracle (flat restatement, oracle/port) to the
reference — its known answers, the committed golden fixtures generated from
the compiled reference, and live byte-for-byte runs of the reference core."""
import json
import math
import tempfile

import numpy as np
import pytest

from cases import static_cases, trace_cases
from oracle_lib import Port, Ref, ref_available
from pathlib import Path

GOLDEN = json.loads((Path(__file__).parent / "golden" / "cases.json").read_text())
CASES = static_cases()


def _row(p):
    return [p[k] for k in ("tau0", "w0", "ws", "tauB", "tauS", "p_max", "kB", "kS")]


# ---- perf model known answers (proj/tests/test_perf_model.cpp) -------------------
def _params(**kw):
    base = dict(tau0=0.0, w0=0.0, ws=1.0, tauB=0.0, tauS=0.0, p_max=1.0, kB=1.0, kS=1.0)
    base.update(kw)
    return _row(base)


@pytest.mark.parametrize("impl", ["port", "ref"])
def test_perf_model_known_answers(impl, port):
    lib = port if impl == "port" else (Ref() if ref_available() else pytest.skip("no ref"))
    # throughput(p{10, kB .5, kS .01}, {2, 100}) — test_perf_model.cpp:43-51
    T, thr = lib.perf_eval(_params(p_max=10.0, kB=0.5, kS=0.01), [2], [100])
    assert thr[0] == pytest.approx(3.995764008937280535437497, rel=1e-13)
    # predict_latency at (1, 1) — :104-117
    T, _ = lib.perf_eval(_params(tau0=1.5, w0=2.0, ws=1.2, tauB=0.3, tauS=0.01, p_max=8.0,
                                 kB=0.7, kS=0.05), [1], [1])
    assert T[0] == pytest.approx(18.10206826697007059858764, rel=1e-13)
    # saturated throughput reduces T to tau0 + S / p_max — :91-102
    T, thr = lib.perf_eval(_params(tau0=5.0, kB=1000.0, kS=1000.0), [4], [100])
    assert T[0] == pytest.approx(105.0, rel=1e-8)
    # strict bound below p_max even in deep saturation — :66-69
    _, thr = lib.perf_eval(_params(p_max=17.0, kB=1000.0, kS=1000.0), [1000000], [1000000000])
    assert thr[0] < 17.0


def test_perf_model_rejects_invalid(port):
    with pytest.raises(ValueError):
        port.perf_eval(_params(), [0], [5])
    with pytest.raises(ValueError):
        port.perf_eval(_params(), [4], [3])
    with pytest.raises(ValueError):
        port.perf_eval(_params(p_max=-1.0), [1], [1])


@pytest.mark.skipif(not ref_available(), reason="reference core not built")
def test_perf_model_port_bitwise_equals_reference(port):
    ref = Ref()
    rng = np.random.default_rng(7)
    for _ in range(20):
        p = _params(tau0=rng.uniform(0, 10), w0=rng.uniform(0, 5), ws=rng.uniform(0.2, 5),
                    tauB=rng.uniform(0, 2), tauS=rng.uniform(0, 0.01),
                    p_max=math.exp(rng.uniform(math.log(0.5), math.log(50))),
                    kB=math.exp(rng.uniform(math.log(0.05), math.log(5))),
                    kS=math.exp(rng.uniform(math.log(1e-4), math.log(0.2))))
        b = rng.integers(1, 1000, 500)
        s = b + rng.integers(0, 100000, 500)
        a = port.perf_eval(p, b, s)
        r = ref.perf_eval(p, b, s)
        assert np.array_equal(a[0], r[0]) and np.array_equal(a[1], r[1])


# ---- the restatement against the pinned golden fixtures -------------------------
@pytest.mark.parametrize("name", sorted(CASES))
def test_port_matches_golden(name, port):
    got = port.run(CASES[name])
    want = GOLDEN[name]
    assert got["event_hash"] == want["event_hash"]
    assert got["arrival_hash"] == want["arrival_hash"]
    assert got["decisions"] == want["decisions"]
    assert got["summary_json"] == want["summary_json"]


def test_port_matches_golden_traces(port):
    from paper_2509_23384_b200 import sim
    with tempfile.TemporaryDirectory() as td:
        for name, cfg in trace_cases(td, sim.synth_generate).items():
            got = port.run(cfg)
            assert got["summary_json"] == GOLDEN[name]["summary_json"], name
            assert got["event_hash"] == GOLDEN[name]["event_hash"], name


# ---- live reference runs on fresh seeds (reference compiled here) ---------------
@pytest.mark.skipif(not ref_available(), reason="reference core not built")
@pytest.mark.parametrize("seed", [21, 22, 23])
@pytest.mark.parametrize("policy", ["prism", "round_robin", "least_loaded", "latency_based",
                                    "weighted", "session_affinity"])
def test_port_matches_reference_live(seed, policy, port):
    from paper_2509_23384_b200 import workloads as W
    cfg = W.sweep_replica(rate=10.0 + 7.5 * (seed - 21), seed=seed, policy=policy, n=250)
    a, b = Ref().run(cfg, records=True), port.run(cfg, records=True)
    for k in ("event_hash", "arrival_hash", "summary_json", "rec_id", "rec_engine", "rec_first",
              "rec_done"):
        assert a[k] == b[k], k


@pytest.mark.skipif(not ref_available(), reason="reference core not built")
def test_port_batch_runner_matches_reference():
    from paper_2509_23384_b200 import workloads as W
    cfgs = W.sweep_configs(8, n=150)
    d1, h1, _ = Ref().run_batch(cfgs, 4)
    d2, h2, _ = Port().run_batch(cfgs, 4)
    assert d1 == d2 and h1 == h2


def test_reference_errors_are_mirrored(port):
    bad = dict(CASES["c1_small"])
    bad = json.loads(json.dumps(bad))
    bad["engines"] = []
    with pytest.raises(RuntimeError):
        port.run(bad)
