"""PRISM router API (mirror of proj/include/servesim/router.h) on K3.

``Router`` keeps the reference's methods (register_engine, on_report,
route, score_affinity, demand_estimate_tokens); every ``route`` runs
nx_route_kernel on the device, and the router's state (report view with
dispatch echoes, session memory, round-robin cursor, weighted RNG) lives
in the same records the batched ``route_batch`` takes. Errors map to the
reference's exceptions: ValueError (invalid_argument), RuntimeError
(runtime_error, e.g. routing with no engines).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import abi
from ._lib import check, lib

POLICIES = {"prism": 0, "round_robin": 1, "session_affinity": 2, "least_loaded": 3,
            "latency_based": 4, "weighted": 5}


@dataclass
class RouterConfig:  # router.h:31-52
    policy: str = "prism"
    weights: tuple = (1.0, 1.0, 1.0, 1.0)
    beta_aff: float = 1.5
    latency_knee: float = 0.5
    latency_scale_ms: float = 0.0
    load_half_ms: float = 50.0
    capacity_headroom: float = 2.0
    staleness_limit_ms: float = 1000.0
    static_weights: dict = field(default_factory=dict)


@dataclass
class RouteDecision:  # router.h:67-72
    engine_id: int = -1
    score: float = 0.0
    factors: tuple = (1.0, 1.0, 1.0, 1.0)
    degraded: bool = False


class Router:
    """servesim::Router (router.cpp:62-289) with device-side route()."""

    def __init__(self, cfg: RouterConfig, ttft_slo_ms: float, rng_state=(1, 2, 3, 4),
                 max_sessions: int = 4096):
        self.cfg = cfg
        self.group = np.zeros(1, dtype=abi.ROUTE_GROUP)
        g = self.group[0]
        g["weights"] = cfg.weights
        g["beta_aff"], g["latency_knee"] = cfg.beta_aff, cfg.latency_knee
        g["latency_scale_ms"], g["load_half_ms"] = cfg.latency_scale_ms, cfg.load_half_ms
        g["capacity_headroom"], g["staleness_limit_ms"] = cfg.capacity_headroom, cfg.staleness_limit_ms
        g["ttft_slo_ms"] = ttft_slo_ms
        g["l_bar_ema"] = 128.0
        g["rng"] = rng_state
        g["policy"] = POLICIES[cfg.policy]
        self.reports = np.zeros(0, dtype=abi.ENGINE_REPORT)
        self.sessions: dict[str, int] = {}
        self.session_map = np.full(max_sessions, -1, dtype=np.int32)

    def register_engine(self, engine_id: int) -> None:
        if engine_id in set(self.reports["engine_id"].tolist()):
            raise ValueError("engine registered twice")
        row = np.zeros(1, dtype=abi.ENGINE_REPORT)
        row["engine_id"] = engine_id
        row["p_max"] = 1.0
        row["static_weight"] = self.cfg.static_weights.get(engine_id, 1.0)
        self.reports = np.concatenate([self.reports, row])

    def on_report(self, engine_id: int, l_hat_ms: float, w_load_tokens: float,
                  m_free_tokens: float, p_max: float, reported_at_ms: float, queue_len: int) -> None:
        idx = np.nonzero(self.reports["engine_id"] == engine_id)[0]
        if idx.size == 0:
            raise ValueError("report from unregistered engine")
        r = self.reports[idx[0]]
        r["l_hat_ms"], r["w_load_tokens"], r["m_free_tokens"] = l_hat_ms, w_load_tokens, m_free_tokens
        r["p_max"], r["reported_at_ms"], r["queue_len"], r["has_report"] = p_max, reported_at_ms, queue_len, 1

    def on_completion(self, engine_id: int, session_id: str, decode_len: int) -> None:
        """router.cpp:83-92 (the latency window of latency_based is not kept)."""
        idx = np.nonzero(self.reports["engine_id"] == engine_id)[0]
        if idx.size == 0:
            return
        g = self.group[0]
        le = g["l_bar_ema"] + 0.05 * (float(decode_len) - g["l_bar_ema"])
        g["l_bar_ema"] = 1.0 if le < 1.0 else le
        self.session_map[self._session(session_id)] = idx[0]

    def _session(self, session_id: str) -> int:
        if session_id not in self.sessions:
            if len(self.sessions) >= self.session_map.size:
                raise ValueError("Router: session table full")
            self.sessions[session_id] = len(self.sessions)
        return self.sessions[session_id]

    def score_affinity(self, engine_id: int, session_id: str) -> float:
        s = self.sessions.get(session_id)
        if s is None or self.session_map[s] < 0:
            return 1.0
        return self.cfg.beta_aff if int(self.reports["engine_id"][self.session_map[s]]) == engine_id else 1.0

    def demand_estimate_tokens(self, prompt_len: int) -> float:
        return max(1.0, float(prompt_len) + float(self.group[0]["l_bar_ema"]))

    def route(self, prompt_len: int, session_id: str, now_ms: float) -> RouteDecision:
        req = np.zeros(1, dtype=abi.ROUTE_REQUEST)
        req["now_ms"], req["prompt_len"], req["session"] = now_ms, prompt_len, self._session(session_id)
        g = self.group[0]
        g["n_engines"], g["n_requests"], g["n_sessions"] = self.reports.size, 1, self.session_map.size
        g["engine_off"] = g["request_off"] = g["session_off"] = 0
        dec, st = route_batch(self.group, self.reports, req, self.session_map)
        d = dec[0]
        return RouteDecision(int(d["engine_id"]), float(d["score"]), tuple(float(x) for x in d["factors"]),
                             bool(d["degraded"]))


def route_batch(groups: np.ndarray, reports: np.ndarray, requests: np.ndarray,
                session_map: np.ndarray, raise_errors: bool = True, mode: int = 0):
    """Batched Router::route on host record arrays (updated in place like the
    routers' own state). Returns (decisions, group_status). mode:
    NX_DETERMINISTIC_FP64 (0, bit-exact) or NX_FAST_FP32 (1, float PRISM
    scores)."""
    for a in (groups, reports, requests, session_map):
        assert a.flags["C_CONTIGUOUS"]
    dec = np.zeros(requests.size, dtype=abi.ROUTE_DECISION)
    st = np.zeros(groups.size, dtype=np.int32)
    rc = lib().nx_prism_route_mode_host(abi.ptr(groups), groups.size, abi.ptr(reports), reports.size,
                                        abi.ptr(requests), requests.size, abi.ptr(session_map),
                                        session_map.size, abi.ptr(dec), abi.ptr(st), mode)
    if raise_errors or not (st != 0).any():
        check(rc)
    return dec, st


def router_rng_state(root_seed: int) -> list:
    """State of the Router's weighted-policy stream, Rng(substream_seed(seed,
    "router")) (router.cpp:62-64)."""
    import ctypes as C
    out = (C.c_uint64 * 4)()
    check(lib().nx_rng_state(root_seed, b"router", 0, out))
    return list(out)
