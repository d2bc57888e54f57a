"""Synthetic workloads for the five BASELINE.json configurations.

Each builder returns a RunConfig JSON dict in the reference's own schema
(proj/src/sim.cpp:454-582 / proj/presets/*.json), so the SAME document drives
the reference simulator (oracle/_ref), the CPU restatement (oracle/_port) and
the device path. Configs 2 and 4 need recorded arrivals (the reference has no
Gamma or long-context generator — SURVEY.md §0.6); `write_gamma_trace` and
`write_longctx_trace` are harness code that writes JSONL traces in the
reference's trace format (proj/src/workload.cpp:83-135), replayed in
``"mode": "timestamp"`` by every arm.
"""
from __future__ import annotations

import json
import math
import os
import random
from pathlib import Path

HET8 = ["fast", "fast", "medium", "medium", "medium", "slow", "slow", "slow"]
SWEEP_RATES = [10.0 + 2.5 * i for i in range(16)]           # 10, 12.5, ..., 47.5 req/s
SWEEP_POLICIES = ["prism", "round_robin", "least_loaded", "latency_based"]


def _engines(profiles, **kw):
    out = []
    for i, p in enumerate(profiles):
        e = {"engine_id": i, "profile": p, "noise_sigma": 0.05, "kv_blocks": 8192,
             "block_size": 16, "scheduler_policy": "lens"}
        e.update(kw)
        out.append(e)
    return out


def config1(seed: int = 1, rate: float = 8.0, n: int = 1000) -> dict:
    """Single fast engine, LENS only, sharegpt Poisson."""
    return {
        "seed": seed, "duration_ms": 3.6e6,
        "slo": {"ttft_slo_ms": 1500, "tpot_slo_ms": 25},
        "router": {"policy": "prism"},
        "engines": _engines(["fast"], kv_blocks=16384),
        "workload": {"scenario": "sharegpt", "mode": "qps", "rate": rate, "n": n,
                     "poisson": True},
    }


def config3(seed: int = 3, rate: float = 40.0, n: int = 100_000, policy: str = "prism") -> dict:
    """8 heterogeneous engines, LENS + PRISM, sharegpt Poisson (§8(d).3)."""
    return {
        "seed": seed, "duration_ms": 3.6e6,
        "slo": {"ttft_slo_ms": 1500, "tpot_slo_ms": 25},
        "router": {"policy": policy},
        "engines": _engines(HET8),
        "workload": {"scenario": "sharegpt", "mode": "qps", "rate": rate, "n": n,
                     "poisson": True},
    }


def sweep_replica(rate: float, seed: int, policy: str, n: int = 2000) -> dict:
    """One replica of the 4096-replica sweep (config 5, §8(d).5)."""
    return config3(seed=seed, rate=rate, n=n, policy=policy)


def sweep_configs(n_replicas: int = 4096, n: int = 2000) -> list[dict]:
    """rate x seed x policy grid; 16 x 64 x 4 = 4096 at full size. Smaller
    counts take an interleaved prefix so every rate and policy is represented."""
    grid = []
    for seed in range(1, 65):
        for rate in SWEEP_RATES:
            for pol in SWEEP_POLICIES:
                grid.append((rate, seed, pol))
    # interleave cost classes: order by seed first so a prefix spans all rates
    return [sweep_replica(r, s, p, n) for (r, s, p) in grid[:n_replicas]]


def _gamma_arrivals(n: int, rate: float, cv: float, seed: int) -> list[float]:
    rng = random.Random(seed)
    shape = 1.0 / (cv * cv)
    scale = (1000.0 / rate) / shape
    t, out = 0.0, []
    for _ in range(n):
        out.append(t)
        t += rng.gammavariate(shape, scale)
    return out


def config2(trace_path: str, seed: int = 2, rate: float = 20.0, n: int = 10_000,
            lengths=None) -> dict:
    """4 homogeneous fast engines, PRISM, bursty Gamma (CV 3) arrivals (§8(d).2).
    `lengths` = (prompts, outputs, sessions) from the reference-equivalent
    synthesizer; the trace file must already exist (see write_trace)."""
    return {
        "seed": seed, "duration_ms": 3.6e6,
        "slo": {"ttft_slo_ms": 1500, "tpot_slo_ms": 25},
        "router": {"policy": "prism"},
        "engines": _engines(["fast"] * 4, kv_blocks=16384),
        "workload": {"trace": trace_path, "mode": "timestamp"},
    }


def config4(trace_path: str, seed: int = 4) -> dict:
    """Long-context mix, 4 heterogeneous engines, kv 65536 blocks (§8(d).4)."""
    return {
        "seed": seed, "duration_ms": 2.0e7,
        "slo": {"ttft_slo_ms": 60000, "tpot_slo_ms": 40},
        "scheduler": {"m_max": 8192, "q_max": 256},
        "router": {"policy": "prism"},
        "engines": _engines(["fast", "fast", "medium", "slow"], kv_blocks=65536),
        "workload": {"trace": trace_path, "mode": "timestamp"},
    }


def baseline_configs(tmpdir, synth) -> dict:
    """BASELINE.json configs 1-4 at their stated sizes:
    1k-request single-engine LENS; 10k-request Gamma CV 3 traces at 20 and
    40 req/s over 4 PRISM engines; 100k requests over 8 heterogeneous
    engines; 2k long-context prompts (8k-128k tokens) over 4 engines with
    65,536 KV blocks. Traces are written under `tmpdir` with `synth` (the
    host synthesiser, reference synth_generate semantics)."""
    g20 = os.path.join(str(tmpdir), "gamma_cv3_r20.jsonl")
    g40 = os.path.join(str(tmpdir), "gamma_cv3_r40.jsonl")
    lc = os.path.join(str(tmpdir), "longctx_2k.jsonl")
    write_gamma_trace(g20, synth, n=10_000, rate=20.0, seed=2)
    write_gamma_trace(g40, synth, n=10_000, rate=40.0, seed=2)
    write_longctx_trace(lc, synth, n=2000, rate=0.5, seed=4)
    return {
        "config1_lens_1k": config1(),
        "config2_gamma_r20_10k": config2(g20, rate=20.0),
        "config2_gamma_r40_10k": config2(g40, rate=40.0),
        "config3_het8_100k": config3(),
        "config4_longctx_2k": config4(lc),
    }


def write_jsonl_trace(path: str | os.PathLike, arrivals, prompts, outputs, sessions) -> None:
    """Reference trace format (workload.cpp:123-135). Python's json emits the
    shortest round-trip repr for floats, so every reader parses the same doubles."""
    with open(path, "w") as f:
        for a, p, o, s in zip(arrivals, prompts, outputs, sessions):
            f.write(json.dumps({"arrival_ms": float(a), "session_id": s,
                                "prompt_tokens": int(p), "output_tokens": int(o)},
                               separators=(",", ":")) + "\n")


def write_gamma_trace(path, synth, n: int = 10_000, rate: float = 20.0, seed: int = 2,
                      cv: float = 3.0) -> None:
    """`synth(scenario, n, seed)` -> (prompts, outputs, sessions) from the
    host synthesizer (reference synth_generate semantics)."""
    prompts, outputs, sessions = synth("sharegpt", n, seed)
    write_jsonl_trace(path, _gamma_arrivals(n, rate, cv, seed), prompts, outputs, sessions)


def write_longctx_trace(path, synth, n: int = 2000, rate: float = 0.5, seed: int = 4) -> None:
    """Prompts log-uniform in [8192, 131072], summarization output lengths,
    Poisson arrivals at `rate`/s."""
    _, outputs, _ = synth("summarization", n, seed)
    rng = random.Random(seed)
    prompts = [int(round(math.exp(rng.uniform(math.log(8192), math.log(131072))))) for _ in range(n)]
    t, arrivals = 0.0, []
    for _ in range(n):
        arrivals.append(t)
        t += rng.expovariate(rate / 1000.0)
    sessions = [f"L{i}" for i in range(n)]
    write_jsonl_trace(path, arrivals, prompts, outputs, sessions)
