"""CPU suite for the product's host side: the C-ABI library loads and exports
every entry point include/nx_sched.h declares; the host front-end (config
parsing, workload synthesis) reproduces the reference's arrival stream and
config errors; the benchmark's replica sharding partitions the sweep."""
import json
import re
import tempfile
from pathlib import Path

import pytest

from cases import static_cases, trace_cases
from oracle_lib import Ref, ref_available
from paper_2509_23384_b200 import _lib, sim, workloads as W

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((ROOT / "tests" / "golden" / "cases.json").read_text())


def declared_symbols():
    text = (ROOT / "include" / "nx_sched.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cuda_device_fails_loudly():
    # With no GPU the product must raise, never fall back to a CPU path.
    if _lib.lib().nx_device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(_lib.CudaError):
        sim.run_simulation(W.config1(n=10))


def test_unknown_evaluation_mode_is_invalid_argument_before_any_device_work():
    # NX_DETERMINISTIC_FP64 / NX_FAST_FP32 only (include/nx_sched.h); checked on
    # the host, so the error class is the same with or without a GPU.
    import numpy as np
    from paper_2509_23384_b200 import abi, lens, router
    probs = np.zeros(1, dtype=abi.LENS_PROBLEM)
    with pytest.raises(ValueError):
        lens.schedule_batch(probs, np.zeros(0, dtype=np.int32), mode=7)
    g = np.zeros(1, dtype=abi.ROUTE_GROUP)
    with pytest.raises(ValueError):
        router.route_batch(g, np.zeros(0, dtype=abi.ENGINE_REPORT), np.zeros(0, dtype=abi.ROUTE_REQUEST),
                           np.zeros(0, dtype=np.int32), mode=3)


@pytest.mark.parametrize("name", sorted(static_cases()))
def test_host_workload_reproduces_reference_arrivals(name):
    h, n, _ = sim.workload_info(static_cases()[name])
    assert f"{h:016x}" == GOLDEN[name]["arrival_hash"]


def test_host_workload_traces_reproduce_reference_arrivals():
    with tempfile.TemporaryDirectory() as td:
        for name, cfg in trace_cases(td, sim.synth_generate).items():
            h, _, _ = sim.workload_info(cfg)
            assert f"{h:016x}" == GOLDEN[name]["arrival_hash"], name


@pytest.mark.parametrize("mutate,exc", [
    (lambda c: c.update(engines=[]), RuntimeError),
    (lambda c: c["workload"].update(rate=0.0), RuntimeError),
    (lambda c: c["workload"].update(mode="timestamp"), RuntimeError),
    (lambda c: c["router"].update(policy="nope"), RuntimeError),
    (lambda c: c["engines"][0].update(scheduler_policy="fifo"), RuntimeError),
    (lambda c: c["engines"].append(dict(c["engines"][0])), RuntimeError),
    (lambda c: c["engines"][0].update(profile="huge"), RuntimeError),
    (lambda c: c["router"].update(weights=[1.0, 2.0]), RuntimeError),
    (lambda c: c["engines"][0].update(true_params={"tau0": -1, "w0": 0, "ws": 1, "tauB": 0,
                                                   "tauS": 0, "p_max": 1, "kB": 1, "kS": 1}),
     ValueError),
])
def test_config_errors_match_reference_exception_class(mutate, exc):
    cfg = json.loads(json.dumps(W.config1(n=20)))
    mutate(cfg)
    with pytest.raises(exc):
        sim.workload_info(cfg)
    if ref_available():  # the reference raises the same class
        with pytest.raises(RuntimeError):
            Ref().run(cfg)


def test_prefill_priority_cap_is_a_runtime_error():
    cfg = W.config1(n=200)
    cfg["engines"][0].update(scheduler_policy="prefill_priority", m_max=128, q_max=64)
    cfg["scheduler"] = {"q_max": 64}
    with pytest.raises(RuntimeError):
        sim.workload_info(cfg)


def test_synth_generate_matches_reference_stream():
    p, o, s = sim.synth_generate("sharegpt", 2000, 3)
    assert min(p) >= 1 and min(o) >= 1
    assert s[0] == "s0" and len(set(s)) < 2000  # follow-up turns reuse live sessions
    # the arrival hash of the same stream is pinned by the golden fixtures above


def test_bench_shards_partition_the_sweep():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    full = W.sweep_configs(64, n=50)
    shards = [bench.shard_configs(r, 16, 50) for r in range(4)]
    flat = [json.dumps(c, sort_keys=True) for sh in shards for c in sh]
    assert flat == [json.dumps(c, sort_keys=True) for c in full]
    rates = {c["workload"]["rate"] for c in shards[0]}
    pols = {c["router"]["policy"] for c in shards[0]}
    assert len(rates) == 4 and len(pols) == 4
