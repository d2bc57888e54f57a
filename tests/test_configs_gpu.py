"""BASELINE.json configs 1-4 at their stated sizes on the device, against the
reference simulator (oracle/_ref) on the same configs and traces.

SURVEY.md §8(d).1-4: 1k-request single-engine LENS; 10k-request Gamma CV 3
traces at 20 and 40 req/s over 4 PRISM engines; 100k requests over 8
heterogeneous engines; 2k long-context prompts (8k-128k tokens, 65,536 KV
blocks). These reach the capacity paths the small parity cases cannot: 128k
prompts against the KV reservation (engine.cpp:184-214), 100k-request
session and queue arenas, 10k-request Gamma bursts.

All five run as ONE device batch; the reference runs each on its own host
thread. Bit-exact: event_hash, arrival_hash, decisions, every RequestRecord,
metrics and engine shares; learner p_max within P_MAX_TOL.
"""
import json
from concurrent.futures import ThreadPoolExecutor

import pytest

from oracle_lib import Port, Ref, ref_available
from test_gpu_parity import assert_same_summary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full_size(tmp_path_factory):
    from paper_2509_23384_b200 import sim, workloads as W
    td = tmp_path_factory.mktemp("baseline_traces")
    cfgs = W.baseline_configs(str(td), sim.synth_generate)
    names = list(cfgs)
    chk = Ref() if ref_available() else Port()
    with ThreadPoolExecutor(max_workers=len(names)) as ex:
        fut = {n: ex.submit(chk.run, cfgs[n], True) for n in names}
        b = sim.Batch([cfgs[n] for n in names]).run()
        want = {n: fut[n].result() for n in names}
    yield names, cfgs, b, want
    b.close()


def test_sizes_are_the_stated_ones(full_size):
    names, cfgs, b, want = full_size
    sums = b.summaries()
    arrived = {n: sums[i].arrived for i, n in enumerate(names)}
    assert arrived == {"config1_lens_1k": 1000, "config2_gamma_r20_10k": 10_000,
                       "config2_gamma_r40_10k": 10_000, "config3_het8_100k": 100_000,
                       "config4_longctx_2k": 2000}
    assert cfgs["config4_longctx_2k"]["engines"][0]["kv_blocks"] == 65536


def test_full_size_bit_exact(full_size):
    names, cfgs, b, want = full_size
    sums = b.summaries()
    for i, n in enumerate(names):
        w = want[n]
        assert sums[i].status == 0, (n, b.error(i))
        assert f"{sums[i].event_hash:016x}" == w["event_hash"], n
        assert sums[i].decisions == w["decisions"], n
        assert_same_summary(w["summary_json"], b.summary_json(i))


def test_full_size_records(full_size):
    names, cfgs, b, want = full_size
    for i, n in enumerate(names):
        w = want[n]
        got = b.records(i)
        assert [r.request_id for r in got] == w["rec_id"], n
        assert [r.engine_id for r in got] == w["rec_engine"], n
        assert [r.first_token_ms for r in got] == w["rec_first"], n
        assert [r.completed_ms for r in got] == w["rec_done"], n
        assert [r.arrival_ms for r in got] == w["rec_arrival"], n


def test_long_context_prompts_reach_the_kv_reservation(full_size):
    """Config 4's prompts span 8k-128k tokens against m_max 8192: most need
    several chunked prefill steps, and a 65,536-block engine holds only a few
    of them at once (KV reservation of the full footprint, engine.cpp:195-201)."""
    names, cfgs, b, want = full_size
    i = names.index("config4_longctx_2k")
    trace = cfgs["config4_longctx_2k"]["workload"]["trace"]
    prompts = [json.loads(line)["prompt_tokens"] for line in open(trace)]
    assert min(prompts) >= 8192 and max(prompts) > 120_000
    assert sum(p > 8192 for p in prompts) > 1000
    s = json.loads(b.summary_json(i))
    assert s["completed"] == json.loads(want["config4_longctx_2k"]["summary_json"])["completed"]
    assert s["completed"] > 0
