"""Parity case catalogue shared by the CPU (port vs reference) and GPU
(device vs reference) suites. Small enough that the reference finishes each
in well under a second, broad enough to reach every branch of the hot path:
all router policies, every engine scheduler policy, KV pressure (trim +
prefix-cache eviction), admission caps, stale reports, recorded-arrival
traces (Gamma bursts, long-context), duration cut-offs and noise-free
engines. Preset-shaped cases restate the values of proj/presets/*.json.
"""
from __future__ import annotations

import copy
import math
import random

from paper_2509_23384_b200 import workloads as W


def _het(n=800, policy="prism", seed=3, rate=40.0, **eng):
    c = W.config3(seed=seed, rate=rate, n=n, policy=policy)
    for e in c["engines"]:
        e.update(eng)
    return c


def static_cases() -> dict:
    cases = {
        "c1_small": W.config1(n=300),
        "c1_low_rate": W.config1(seed=2, rate=4.0, n=300),
        "het_prism": _het(1200),
        "het_round_robin": _het(800, "round_robin"),
        "het_least_loaded": _het(800, "least_loaded"),
        "het_latency_based": _het(800, "latency_based"),
        "het_weighted": _het(800, "weighted"),
        "het_session_affinity": _het(800, "session_affinity"),
        "prefill_priority": _het(500, scheduler_policy="prefill_priority"),
        "static_chunked": _het(500, scheduler_policy="static_chunked", static_budget=512),
        "wait_cap": _het(600, rate=80.0, wait_cap=3),
        "kv_pressure": _het(500, rate=60.0, kv_blocks=384),
        "noise_free": _het(400, noise_sigma=0.0),
        "sweep_low_rate": W.sweep_replica(10.0, 5, "least_loaded", n=400),
        "sweep_high_rate": W.sweep_replica(47.5, 6, "latency_based", n=400),
    }
    mixed = _het(500)
    for i, e in enumerate(mixed["engines"]):
        e["scheduler_policy"] = ["lens", "prefill_priority", "static_chunked"][i % 3]
        e["static_budget"] = 256 + 128 * i
    cases["mixed_policies"] = mixed
    cut = _het(800)
    cut["duration_ms"] = 7000.0
    cases["duration_cutoff"] = cut
    stale = _het(600, state_report_period_ms=400.0, state_staleness_ms=1100.0)
    stale["router"].update({"staleness_limit_ms": 500.0})
    cases["stale_reports"] = stale
    # heterogeneous4.json-shaped (static weights, 1 s reports, 250 ms staleness)
    h4 = {
        "seed": 4, "duration_ms": 3000000.0, "slo": {"ttft_slo_ms": 1500, "tpot_slo_ms": 25},
        "scheduler": {"m_max": 8192, "q_max": 256, "n_search_iters": 10, "eps_ratio": 0.05, "q_ref": 16},
        "learner": {"long_window": 4096, "short_window": 64, "structural_period": 64,
                    "linear_period": 16, "min_structural_samples": 64},
        "router": {"policy": "prism", "weights": [1.0, 1.0, 1.0, 1.0], "beta_aff": 1.2,
                   "latency_knee": 0.5, "load_half_ms": 150, "capacity_headroom": 2.0,
                   "staleness_limit_ms": 1000, "latency_window_ms": 2000,
                   "static_weights": {"0": 4.0, "1": 2.0, "2": 2.0, "3": 1.0}},
        "engines": [{"engine_id": i, "profile": p, "noise_sigma": 0.05, "kv_blocks": kv,
                     "block_size": 16, "scheduler_policy": "lens",
                     "state_report_period_ms": 1000, "state_staleness_ms": 250}
                    for i, (p, kv) in enumerate([("fast", 8192), ("medium", 6144),
                                                 ("medium", 6144), ("slow", 4096)])],
        "workload": {"scenario": "sharegpt", "mode": "qps", "rate": 26, "n": 700},
    }
    cases["preset_heterogeneous4"] = h4
    h4w = copy.deepcopy(h4)
    h4w["router"]["policy"] = "weighted"
    cases["preset_heterogeneous4_weighted"] = h4w
    # homogeneous8.json-shaped (flowgpt, tight TPOT)
    cases["preset_homogeneous8"] = {
        "seed": 4, "duration_ms": 600000, "slo": {"ttft_slo_ms": 1500, "tpot_slo_ms": 12},
        "router": {"policy": "prism"},
        "engines": [{"engine_id": i, "profile": "fast", "noise_sigma": 0.05, "kv_blocks": 16384,
                     "block_size": 16, "scheduler_policy": "lens"} for i in range(8)],
        "workload": {"scenario": "flowgpt", "mode": "qps", "rate": 8.0, "n": 300},
        "learner": {"long_window": 4096, "short_window": 64, "structural_period": 64,
                    "linear_period": 16, "min_structural_samples": 64},
    }
    # summarization_lens.json / zeroconfig.json-shaped
    cases["preset_summarization_lens"] = {
        "seed": 2, "duration_ms": 3000000.0, "slo": {"ttft_slo_ms": 2000, "tpot_slo_ms": 10},
        "learner": {"long_window": 4096, "short_window": 64, "structural_period": 256,
                    "linear_period": 32, "min_structural_samples": 128},
        "router": {"policy": "round_robin"},
        "engines": [{"engine_id": 0, "profile": "fast", "noise_sigma": 0.05, "kv_blocks": 24576,
                     "block_size": 16, "scheduler_policy": "lens", "static_budget": 512}],
        "workload": {"scenario": "summarization", "mode": "qps", "rate": 1.125, "n": 120},
    }
    cases["preset_zeroconfig"] = {
        "seed": 1, "duration_ms": 120000, "slo": {"ttft_slo_ms": 1500, "tpot_slo_ms": 25},
        "learner": {"long_window": 4096, "short_window": 64, "structural_period": 192,
                    "linear_period": 16, "min_structural_samples": 128},
        "router": {"policy": "round_robin"},
        "engines": [{"engine_id": 0, "profile": "medium", "noise_sigma": 0.05,
                     "kv_blocks": 16384, "block_size": 16, "scheduler_policy": "lens"}],
        "workload": {"scenario": "sharegpt", "mode": "qps", "rate": 6.0, "n": 900},
    }
    # explicit true_params + engine ids out of order + coding scenario
    tp = {"engine_id": 7, "true_params": {"tau0": 3.0, "w0": 12.0, "ws": 1.1, "tauB": 0.05,
                                         "tauS": 0.0002, "p_max": 30.0, "kB": 2.0, "kS": 0.01},
          "noise_sigma": 0.08, "kv_blocks": 6000, "block_size": 32}
    cases["custom_engines"] = {
        "seed": 11, "slo": {"ttft_slo_ms": 1200, "tpot_slo_ms": 30},
        "tradeoff": {"l_bar": 64.0, "td_min_ms": 3.0},
        "router": {"policy": "prism", "latency_scale_ms": 300.0, "weights": [1.0, 2.0, 0.5, 1.0]},
        "engines": [tp, {"engine_id": 2, "profile": "slow"}, {"engine_id": 5, "profile": "fast",
                                                            "m_max": 4096, "q_max": 64}],
        "workload": {"scenario": "coding", "mode": "qps", "rate": 12.0, "n": 500},
    }
    return cases


def trace_cases(tmpdir, synth) -> dict:
    """Configs replaying recorded arrivals (the reference has no Gamma or
    long-context generator). `synth(scenario, n, seed)` is the host
    synthesiser (reference synth_generate semantics)."""
    g = f"{tmpdir}/gamma.jsonl"
    W.write_gamma_trace(g, synth, n=1500, rate=40.0, seed=2)
    lc = f"{tmpdir}/longctx.jsonl"
    W.write_longctx_trace(lc, synth, n=50, rate=0.5, seed=4)
    unsorted = f"{tmpdir}/unsorted.jsonl"
    rng = random.Random(9)
    arr = [rng.uniform(0, 20000.0) for _ in range(300)]
    p, o, s = synth("coding", 300, 9)
    W.write_jsonl_trace(unsorted, arr, p, o, s)
    scaled = W.config2(unsorted)
    scaled["workload"]["time_scale"] = 1.7
    qps = W.config2(g)
    qps["workload"] = {"trace": g, "mode": "qps", "rate": 25.0, "poisson": True}
    return {
        "config2_gamma_cv3": W.config2(g),
        "config4_longctx": W.config4(lc),
        "trace_unsorted_scaled": scaled,
        "trace_qps_reassigned": qps,
    }
