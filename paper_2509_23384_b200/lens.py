"""LENS scheduler API (mirror of proj/include/servesim/lens.h) on K2.

``schedule_step`` keeps the reference signature — wait/run queues of
requests, SLOSpec, TradeoffModel, PerfParams, SchedulerConfig — and returns
a ``BatchPlan`` with the reference's allocations. ``schedule_batch`` is the
batched form: many independent decisions in one launch of nx_lens_kernel
(one warp per decision). Invalid inputs raise ValueError like the
reference's std::invalid_argument (lens.cpp:12-14, 36-38, 96-99).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import abi
from ._lib import NX_DETERMINISTIC_FP64, NX_FAST_FP32, check, lib  # noqa: F401 (mode constants re-exported)
from .perf_model import PerfParams, _row


@dataclass
class SLOSpec:  # lens.h:14-19
    ttft_slo_ms: float = 2000.0
    tpot_slo_ms: float = 12.0


@dataclass
class TradeoffModel:  # lens.h:22-38
    alpha_ms: float = 2000.0
    beta: float = 16.0
    l_bar: float = 128.0
    td_min_ms: float = 2.0

    @staticmethod
    def initial_for(slo: SLOSpec) -> "TradeoffModel":
        return TradeoffModel(2.0 * slo.ttft_slo_ms, slo.ttft_slo_ms / slo.tpot_slo_ms)


@dataclass
class SchedulerConfig:  # lens.h:63-75
    m_max: int = 8192
    q_max: int = 256
    n_search_iters: int = 10
    eps_ratio: float = 0.05
    q_ref: float = 16.0


@dataclass
class Request:  # the fields schedule_step reads (lens.h:41-61)
    id: int = 0
    prompt_len: int = 1
    prefilled: int = 0

    def remaining_prompt(self) -> int:
        return self.prompt_len - self.prefilled


@dataclass
class Allocation:  # lens.h:77-81
    request_id: int
    tokens: int
    is_prefill: bool


@dataclass
class BatchPlan:  # lens.h:82-91
    allocations: list = field(default_factory=list)
    b: int = 0
    s: int = 0
    predicted_ms: float = 0.0
    target_ms: float = 0.0
    overload: bool = False
    slo_risk: bool = False

    def empty(self) -> bool:
        return not self.allocations


def problem_record(n_run: int, n_wait: int, wait_off: int, slo: SLOSpec, tm: TradeoffModel,
                   params, cfg: SchedulerConfig) -> np.ndarray:
    """One nx_lens_problem record."""
    r = np.zeros((), dtype=abi.LENS_PROBLEM)
    r["params"] = _row(params)
    r["ttft_slo_ms"], r["tpot_slo_ms"] = slo.ttft_slo_ms, slo.tpot_slo_ms
    r["alpha_ms"], r["beta"], r["l_bar"], r["td_min_ms"] = tm.alpha_ms, tm.beta, tm.l_bar, tm.td_min_ms
    r["eps_ratio"], r["q_ref"] = cfg.eps_ratio, cfg.q_ref
    r["m_max"], r["q_max"], r["n_search_iters"] = cfg.m_max, cfg.q_max, cfg.n_search_iters
    r["n_run"], r["n_wait"], r["wait_off"] = n_run, n_wait, wait_off
    return r


def schedule_batch(problems: np.ndarray, wait_remaining: np.ndarray, raise_errors: bool = True,
                   mode: int = NX_DETERMINISTIC_FP64):
    """Batched schedule_step on host arrays (copies in/out included).

    problems: nx_lens_problem records; wait_remaining: int32 remaining
    prompts, CSR by problems["wait_off"/"n_wait"]. Returns (plans,
    alloc_tokens) — plans are nx_lens_plan records; alloc_tokens[wait_off+k]
    holds waiter k's prefill chunk for k < n_prefill. With raise_errors
    False, failing problems only report their status in the plan. mode:
    NX_DETERMINISTIC_FP64 (bit-exact) or NX_FAST_FP32 (float probes).
    """
    problems = np.ascontiguousarray(problems, dtype=abi.LENS_PROBLEM)
    rem = np.ascontiguousarray(wait_remaining, dtype=np.int32)
    plans = np.zeros(problems.size, dtype=abi.LENS_PLAN)
    alloc = np.zeros(rem.size, dtype=np.int32)
    rc = lib().nx_lens_schedule_mode_host(abi.ptr(problems), problems.size, abi.ptr(rem), rem.size,
                                          abi.ptr(plans), abi.ptr(alloc), mode)
    if raise_errors or not (plans["status"] != 0).any():
        check(rc)  # per-problem failures leave every plan written (status field)
    return plans, alloc


def schedule_batch_device(problems, wait_remaining, plans, alloc_tokens, stream=None,
                          mode: int = NX_DETERMINISTIC_FP64):
    """Stream-ordered batched schedule_step on torch CUDA tensors (uint8
    views of the record arrays for problems/plans, int32 for the waiters)."""
    st = stream.cuda_stream if stream is not None else None
    check(lib().nx_lens_schedule_mode_dev(problems.data_ptr(), problems.numel() // abi.LENS_PROBLEM.itemsize,
                                          wait_remaining.data_ptr(), wait_remaining.numel(),
                                          plans.data_ptr(), alloc_tokens.data_ptr(), mode, st))


# ---- baseline engine policies (engine.h:68-79) -------------------------------------
PREFILL_PRIORITY, STATIC_CHUNKED = 1, 2   # NX_SCHED_* (SchedulerPolicy order)


def baseline_record(policy: int, n_run: int, n_wait: int, wait_off: int, params, m_max: int = 8192,
                    q_max: int = 256, static_budget: int = 2048, engine_id: int = 0) -> np.ndarray:
    """One nx_baseline_problem record (policy 0 = lens is a logic error)."""
    r = np.zeros((), dtype=abi.BASELINE_PROBLEM)
    r["params"] = _row(params)
    r["m_max"], r["q_max"], r["static_budget"] = m_max, q_max, static_budget
    r["policy"], r["engine_id"] = policy, engine_id
    r["n_run"], r["n_wait"], r["wait_off"] = n_run, n_wait, wait_off
    return r


def schedule_baseline_batch(problems: np.ndarray, wait_remaining: np.ndarray, raise_errors: bool = True):
    """Batched schedule_baseline (engine.cpp:61-108) on host arrays. Returns
    (problems with b/s/predicted_ms/n_decode/n_prefill/status filled,
    tokens) — tokens[wait_off + k] is waiter k's prefill for k < n_prefill."""
    probs = np.array(problems, dtype=abi.BASELINE_PROBLEM, copy=True).reshape(-1)
    rem = np.ascontiguousarray(wait_remaining, dtype=np.int32)
    tok = np.zeros(rem.size, dtype=np.int32)
    rc = lib().nx_baseline_schedule_host(abi.ptr(probs), probs.size, abi.ptr(rem), rem.size, abi.ptr(tok))
    if raise_errors or not (probs["status"] != 0).any():
        check(rc)
    return probs, tok


def schedule_baseline(policy: int, wait_q, run_q, params, m_max: int = 8192, q_max: int = 256,
                      static_budget: int = 2048, engine_id: int = 0) -> BatchPlan:
    """servesim::schedule_baseline (engine.cpp:61-108), one decision on the device."""
    rem = np.asarray([r.remaining_prompt() for r in wait_q], dtype=np.int64)
    if rem.size and (rem.min() < 1 or rem.max() >= 2 ** 31):
        raise ValueError("schedule_baseline: device path needs 1 <= remaining prompt < 2^31")
    prob = baseline_record(policy, len(run_q), len(wait_q), 0, params, m_max, q_max, static_budget, engine_id)
    p, tok = schedule_baseline_batch(prob, rem.astype(np.int32))
    p = p[0]
    plan = BatchPlan(b=int(p["b"]), s=int(p["s"]), predicted_ms=float(p["predicted_ms"]))
    plan.allocations = [Allocation(run_q[i].id, 1, False) for i in range(int(p["n_decode"]))]
    plan.allocations += [Allocation(wait_q[k].id, int(tok[k]), True) for k in range(int(p["n_prefill"]))]
    return plan


def schedule_step(wait_q, run_q, slo: SLOSpec, tm: TradeoffModel, params,
                  cfg: SchedulerConfig) -> BatchPlan:
    """servesim::schedule_step (lens.cpp:96-146), one decision on the device."""
    rem = np.asarray([r.remaining_prompt() for r in wait_q], dtype=np.int64)
    if rem.size and (rem.min() < 1 or rem.max() >= 2 ** 31):
        raise ValueError("schedule_step: device path needs 1 <= remaining prompt < 2^31")
    prob = problem_record(len(run_q), len(wait_q), 0, slo, tm, params, cfg).reshape(1)
    plans, alloc = schedule_batch(prob, rem.astype(np.int32))
    p = plans[0]
    plan = BatchPlan(b=int(p["b"]), s=int(p["s"]), predicted_ms=float(p["predicted_ms"]),
                     target_ms=float(p["target_ms"]), overload=bool(p["overload"]),
                     slo_risk=bool(p["slo_risk"]))
    plan.allocations = [Allocation(run_q[i].id, 1, False) for i in range(int(p["n_decode"]))]
    plan.allocations += [Allocation(wait_q[k].id, int(alloc[k]), True)
                         for k in range(int(p["n_prefill"]))]
    return plan
