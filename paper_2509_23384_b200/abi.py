"""numpy record layouts of the C-ABI structs in include/nx_sched.h.

Batched calls pass arrays of these records straight to the library (zero
copy); ``check_layouts`` compares every itemsize with the C ``sizeof``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import lib

LENS_PROBLEM = np.dtype([
    ("params", "f8", 8), ("ttft_slo_ms", "f8"), ("tpot_slo_ms", "f8"), ("alpha_ms", "f8"),
    ("beta", "f8"), ("l_bar", "f8"), ("td_min_ms", "f8"), ("eps_ratio", "f8"), ("q_ref", "f8"),
    ("m_max", "i8"), ("q_max", "i8"), ("n_search_iters", "i4"), ("n_run", "i4"),
    ("n_wait", "i4"), ("pad_", "i4"), ("wait_off", "i8")], align=True)

LENS_PLAN = np.dtype([
    ("b", "i8"), ("s", "i8"), ("predicted_ms", "f8"), ("target_ms", "f8"), ("overload", "i4"),
    ("slo_risk", "i4"), ("n_decode", "i4"), ("n_prefill", "i4"), ("status", "i4"),
    ("pad_", "i4")], align=True)

ROUTE_GROUP = np.dtype([
    ("weights", "f8", 4), ("beta_aff", "f8"), ("latency_knee", "f8"), ("latency_scale_ms", "f8"),
    ("load_half_ms", "f8"), ("capacity_headroom", "f8"), ("staleness_limit_ms", "f8"),
    ("ttft_slo_ms", "f8"), ("l_bar_ema", "f8"), ("rng", "u8", 4), ("rr_next", "u8"),
    ("policy", "i4"), ("n_engines", "i4"), ("engine_off", "i8"), ("request_off", "i8"),
    ("session_off", "i8"), ("n_requests", "i4"), ("n_sessions", "i4")], align=True)

ENGINE_REPORT = np.dtype([
    ("l_hat_ms", "f8"), ("w_load_tokens", "f8"), ("m_free_tokens", "f8"), ("p_max", "f8"),
    ("reported_at_ms", "f8"), ("static_weight", "f8"), ("queue_len", "i8"), ("engine_id", "i4"),
    ("has_report", "i4"), ("rolling_latency_ms", "f8")], align=True)

ROUTE_REQUEST = np.dtype([("now_ms", "f8"), ("prompt_len", "i8"), ("session", "i4"),
                          ("pad_", "i4")], align=True)

ROUTE_DECISION = np.dtype([("score", "f8"), ("factors", "f8", 4), ("engine_id", "i4"),
                           ("degraded", "i4")], align=True)

REFIT_PROBLEM = np.dtype([
    ("params", "f8", 8), ("long_window", "i8"), ("short_window", "i8"),
    ("min_structural_samples", "i8"), ("sample_off", "i8"), ("n_samples", "i4"),
    ("pad_", "i4")], align=True)

REFIT_RESULT = np.dtype([("params", "f8", 8), ("counters", "i8", 7), ("updated", "i4"),
                         ("status", "i4")], align=True)

BASELINE_PROBLEM = np.dtype([
    ("params", "f8", 8), ("m_max", "i8"), ("q_max", "i8"), ("static_budget", "i8"),
    ("wait_off", "i8"), ("policy", "i4"), ("engine_id", "i4"), ("n_run", "i4"), ("n_wait", "i4"),
    ("b", "i8"), ("s", "i8"), ("predicted_ms", "f8"), ("n_decode", "i4"), ("n_prefill", "i4"),
    ("status", "i4"), ("pad_", "i4")], align=True)

# position in nx_abi_sizes' list -> layout (8, 9: replica summary / request record)
ORDER = {0: LENS_PROBLEM, 1: LENS_PLAN, 2: ROUTE_GROUP, 3: ENGINE_REPORT, 4: ROUTE_REQUEST,
         5: ROUTE_DECISION, 6: REFIT_PROBLEM, 7: REFIT_RESULT, 10: BASELINE_PROBLEM}


def check_layouts() -> None:
    out = (C.c_int64 * 11)()
    lib().nx_abi_sizes(out, 11)
    for i, dt in ORDER.items():
        if dt.itemsize != out[i]:
            raise RuntimeError(f"ABI layout mismatch for struct #{i}: numpy {dt.itemsize} vs C {out[i]}")


def ptr(a) -> int | None:
    """Host data pointer of a contiguous numpy array (None for empty)."""
    if a is None or a.size == 0:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data
