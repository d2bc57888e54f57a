"""The reference's own unit tests — proj/tests/test_perf_model.cpp,
test_lens.cpp, test_router.cpp, test_learner.cpp, test_metrics.cpp,
test_workload.cpp, test_sim.cpp and test_engine.cpp (all 128 cases),
compiled UNMODIFIED (tests/refsuite/Makefile) against the C++ drop-in
include/nx_servesim.hpp — run on the device path: every throughput /
predict_latency, schedule_step, binary_search_budget, allocate_tokens,
target_latency, Router::route, score_*, OnlineLearner refit and
run_simulation / sweep they exercise is a launch of the sm_100a kernels."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent / "refsuite" / "_bin" / "refsuite"


def test_reference_unit_suites_pass_on_the_device_path():
    if not BIN.exists():
        pytest.fail(f"{BIN} not built (python -c 'import __graft_entry__ as g; g.build()')")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=1500)
    summary = [l for l in r.stdout.splitlines() if l.startswith("test cases:")]
    failed = [l for l in r.stdout.splitlines() if l.startswith("[FAIL]")]
    assert summary, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.returncode == 0 and not failed, "\n".join(failed) + "\n" + r.stderr[-4000:]
