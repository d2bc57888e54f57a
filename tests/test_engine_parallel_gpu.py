"""Engine-parallel event loop (device/sim_kernel.cu) against the reference on
the cases that stress its machinery rather than the models:

* more engines than engine warps (engines share warps: 12 and 31 engines);
* every engine-warp count from 1 to 8 giving the same bits (NX_ENGINE_WARPS);
* equal-time events across engines, where the reference's sequence numbers
  decide the order: state-report chains with equal periods (every report of
  every engine ties), staleness equal to the period (a delivery ties with the
  next report), noise-free identical engines under round robin (step
  completions tie);
* the drain rule (sim.cpp:295-300) when arrivals run past the duration and
  when the first arrival is already past it.

Each case is checked against the compiled reference (oracle/_ref, or the
restatement where it is absent): event hash, decisions, every record,
summary. SURVEY.md §8(a) rows a13/a21; the reference's order is sim.cpp:50-55.
"""
import copy
import os

import pytest

from oracle_lib import Port, Ref, ref_available
from test_gpu_parity import assert_same_summary

pytestmark = pytest.mark.gpu


def _checker():
    return Ref() if ref_available() else Port()


def _base(n=300, rate=30.0, policy="prism", seed=5):
    from paper_2509_23384_b200 import workloads as W
    return W.config3(seed=seed, rate=rate, n=n, policy=policy)


def _many_engines(k: int, policy="prism"):
    c = _base(n=400, rate=60.0, policy=policy)
    src = c["engines"]
    c["engines"] = []
    for i in range(k):
        e = copy.deepcopy(src[i % len(src)])
        e["engine_id"] = 100 + 7 * i  # ids need not be dense or ordered like indices
        c["engines"].append(e)
    return c


def _equal_period_reports():
    c = _base(n=300, rate=25.0)
    for e in c["engines"]:
        e["state_report_period_ms"] = 50.0
        e["state_staleness_ms"] = 50.0  # each delivery ties with the next report
    return c


def _mixed_period_reports():
    c = _base(n=300, rate=25.0, policy="least_loaded")
    for i, e in enumerate(c["engines"]):
        e["state_report_period_ms"] = [40.0, 60.0, 80.0][i % 3]
        e["state_staleness_ms"] = [0.0, 40.0, 120.0][i % 3]
    return c


def _noise_free_twins():
    c = _base(n=300, rate=40.0, policy="round_robin")
    for e in c["engines"]:
        e["profile"] = "fast"
        e["noise_sigma"] = 0.0
    return c


def _past_duration():
    c = _base(n=300, rate=20.0)
    c["duration_ms"] = 4000.0  # most arrivals never happen; reports run to the end
    return c


def _nothing_arrives():
    c = _base(n=50, rate=1.0)
    c["duration_ms"] = 0.5  # the first arrival is past the duration
    return c


CASES = {
    "engines_12": lambda: _many_engines(12),
    "engines_31_rr": lambda: _many_engines(31, "round_robin"),
    "equal_period_reports": _equal_period_reports,
    "mixed_period_reports": _mixed_period_reports,
    "noise_free_twins": _noise_free_twins,
    "past_duration": _past_duration,
    "nothing_arrives": _nothing_arrives,
}


@pytest.fixture(scope="module")
def reference():
    chk = _checker()
    cfgs = {n: f() for n, f in CASES.items()}
    return cfgs, {n: chk.run(cfgs[n], True) for n in cfgs}


def _assert_same(b, i, name, want):
    s = b.summaries()[i]
    assert s.status == 0, (name, b.error(i))
    assert f"{s.event_hash:016x}" == want["event_hash"], name
    assert s.decisions == want["decisions"], name
    assert_same_summary(want["summary_json"], b.summary_json(i))
    got = b.records(i)
    assert [r.request_id for r in got] == want["rec_id"], name
    assert [r.completed_ms for r in got] == want["rec_done"], name
    assert [r.first_token_ms for r in got] == want["rec_first"], name


def test_stress_cases_bit_exact(reference):
    from paper_2509_23384_b200 import sim
    cfgs, want = reference
    names = list(cfgs)
    b = sim.Batch([cfgs[n] for n in names]).run()
    for i, n in enumerate(names):
        _assert_same(b, i, n, want[n])
    b.close()


@pytest.mark.parametrize("warps", [1, 3, 5, 8])
def test_engine_warp_count_does_not_change_results(reference, warps, monkeypatch):
    """Engines of one warp run one after another, of different warps side by
    side: the results are the reference's for every split."""
    from paper_2509_23384_b200 import sim
    cfgs, want = reference
    names = ["engines_12", "equal_period_reports", "noise_free_twins"]
    monkeypatch.setenv("NX_ENGINE_WARPS", str(warps))
    b = sim.Batch([cfgs[n] for n in names]).run()
    for i, n in enumerate(names):
        _assert_same(b, i, n, want[n])
    b.close()


def test_more_than_31_engines_is_rejected():
    from paper_2509_23384_b200 import sim
    c = _many_engines(32)
    with pytest.raises(ValueError, match="31 engines"):
        sim.Batch([c])


def test_ties_happen(reference):
    """The tie cases do produce equal-time events across engines (else they
    would not test the order): in the reference's routing log equal-period
    reports make every engine's report land on the same instants."""
    cfgs, want = reference
    s = want["equal_period_reports"]
    assert s["decisions"] > 0
    periods = {e["state_report_period_ms"] for e in cfgs["equal_period_reports"]["engines"]}
    assert periods == {50.0}
    twins = {(e["profile"], e["noise_sigma"]) for e in cfgs["noise_free_twins"]["engines"]}
    assert twins == {("fast", 0.0)}
