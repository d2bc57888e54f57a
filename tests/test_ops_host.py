"""CPU suite for the batched operators' host side: ABI layouts, the golden
fixtures' provenance (regenerated inputs hash to the recorded digests; the
compiled reference reproduces every recorded output), and argument
validation that happens before any device work."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import ops_cases
from oracle_lib import Ref, ref_available

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "ops_golden.json").read_text())
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import make_ops_golden as M  # noqa: E402


def test_abi_layouts_match_c():
    from paper_2509_23384_b200 import abi
    abi.check_layouts()


def test_golden_inputs_regenerate_identically():
    assert M.digest(ops_cases.lens_cases()) == GOLD["digest"]["lens"]
    assert M.digest(ops_cases.route_cases()) == GOLD["digest"]["route"]
    assert M.digest(ops_cases.refit_cases()) == GOLD["digest"]["refit"]
    assert M.digest(ops_cases.baseline_cases()) == GOLD["digest"]["baseline"]


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
def test_reference_reproduces_lens_golden():
    ref = Ref()
    for c, want in zip(ops_cases.lens_cases(), GOLD["lens"]):
        r = ref.schedule_step(c["n_run"], c["prompt"], c["prefilled"], c["ttft"], c["tpot"], c["tm"],
                              c["params"], c["m_max"], c["q_max"], c["n_iters"], c["eps"], c["q_ref"])
        assert r["status"] == want["status"]
        if r["status"] == 0:
            assert r["predicted"].hex() == want["predicted"] and r["b"] == want["b"]
            assert [list(a) for a in r["alloc"]] == want["alloc"]


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
def test_reference_reproduces_route_and_refit_golden():
    ref = Ref()
    for c, want in list(zip(ops_cases.route_cases(), GOLD["route"]))[:40]:
        r = ref.route_group(c["policy"], c["cfg9"], c["ttft"], c["tpot"], c["seed"], c["ids"],
                            c["static_w"], c["states5"], c["qlen"], c["has_report"], c["comp_engine"],
                            c["comp_session"], c["comp_decode"], c["req_prompt"], c["req_session"],
                            c["req_now"])
        assert r["engine"].tolist() == want["engine"]
    metas, b, s, y = ops_cases.refit_cases()
    for m, want in list(zip(metas, GOLD["refit"]))[-20:]:
        sl = slice(m["off"], m["off"] + m["n"])
        r = ref.learner_refit(m["kind"], m["priors"], m["long_w"], m["short_w"], m["min_s"],
                              b[sl], s[sl], y[sl])
        assert r["status"] == want["status"]
        if r["status"] == 0:
            assert [x.hex() for x in r["params"]] == want["params"]


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
def test_reference_reproduces_baseline_golden():
    ref = Ref()
    for c, want in zip(ops_cases.baseline_cases(), GOLD["baseline"]):
        r = ref.schedule_baseline(c["policy"], c["n_run"], c["prompt"], c["prefilled"], c["params"],
                                  c["m_max"], c["q_max"], c["static_budget"], c["engine_id"])
        assert r["status"] == want["status"]
        if r["status"] == 0:
            assert r["predicted"].hex() == want["predicted"] and r["s"] == want["s"]
            assert [list(a) for a in r["alloc"]] == want["alloc"]


def test_host_validation_precedes_device_work():
    from paper_2509_23384_b200 import abi, learner, lens
    probs = np.zeros(1, dtype=abi.LENS_PROBLEM)
    probs["n_wait"], probs["wait_off"] = 5, 0          # 5 waiters, only 2 given
    with pytest.raises(ValueError):
        lens.schedule_batch(probs, np.ones(2, dtype=np.int32))
    rp = np.zeros(1, dtype=abi.REFIT_PROBLEM)
    rp["n_samples"], rp["sample_off"], rp["long_window"] = 10, 0, 64
    with pytest.raises(ValueError):
        learner.refit_batch(learner.LINEAR, rp, [1] * 3, [1] * 3, [1.0] * 3)
    bp = lens.baseline_record(lens.STATIC_CHUNKED, 0, 4, 0, ops_cases.FAST)
    with pytest.raises(ValueError):
        lens.schedule_baseline_batch(bp, np.ones(2, dtype=np.int32))


REFSUITE = ROOT / "tests" / "refsuite" / "_bin" / "refsuite"


@pytest.mark.skipif(not REFSUITE.exists(), reason="refsuite not built (needs /root/reference)")
@pytest.mark.parametrize("suite", ["test_metrics.cpp", "test_workload.cpp"])
def test_reference_host_suites_pass_against_the_drop_in(suite):
    """The reference's metrics and workload unit tests (host-side functions in
    the drop-in: summarize, percentile, write_requests_csv, synth_generate,
    assign_arrivals, trace I/O) compiled unchanged against nx_servesim.hpp."""
    import subprocess
    r = subprocess.run([str(REFSUITE), suite], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "0 failed" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_batched_operators_fail_loudly_without_a_device():
    """No CPU path behind the operators: without a GPU they raise CudaError."""
    from paper_2509_23384_b200 import _lib, abi, lens
    if _lib.lib().nx_device_count() > 0:
        pytest.skip("a CUDA device is present")
    probs = np.zeros(1, dtype=abi.LENS_PROBLEM)
    probs[0] = lens.problem_record(1, 1, 0, lens.SLOSpec(), lens.TradeoffModel(), ops_cases.FAST,
                                   lens.SchedulerConfig())
    with pytest.raises(_lib.CudaError):
        lens.schedule_batch(probs, np.ones(1, dtype=np.int32))
