"""Online-learner refits (mirror of proj/include/servesim/learner.h) on K4.

``refit_batch`` runs OnlineLearner::update_linear or update_structural on
many explicit sample windows at once (nx_refit_kernel, one warp per
learner) — the same device code the simulator's learners use.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import abi
from ._lib import check, lib
from .perf_model import _row

LINEAR, STRUCTURAL = 0, 1
COUNTERS = ("linear_updates", "structural_updates", "degenerate_updates", "rescale_updates",
            "clamp_events", "failed_fits", "low_identifiability")


@dataclass
class LearnerConfig:  # learner.h:12-24
    long_window: int = 4096
    short_window: int = 64
    structural_period: int = 1024
    linear_period: int = 32
    min_structural_samples: int = 256


def problem_record(params, cfg: LearnerConfig, sample_off: int, n_samples: int) -> np.ndarray:
    r = np.zeros((), dtype=abi.REFIT_PROBLEM)
    r["params"] = _row(params)
    r["long_window"], r["short_window"] = cfg.long_window, cfg.short_window
    r["min_structural_samples"] = cfg.min_structural_samples
    r["sample_off"], r["n_samples"] = sample_off, n_samples
    return r


def refit_batch(kind: int, problems: np.ndarray, b, s, y, raise_errors: bool = True) -> np.ndarray:
    """Batched update_linear (kind 0) / update_structural (kind 1) on host
    arrays; samples CSR by problems["sample_off"/"n_samples"], chronological.
    Returns nx_refit_result records (params after, counter increments,
    updated flag)."""
    problems = np.ascontiguousarray(problems, dtype=abi.REFIT_PROBLEM)
    b = np.ascontiguousarray(b, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(problems.size, dtype=abi.REFIT_RESULT)
    rc = lib().nx_refit_host(kind, abi.ptr(problems), problems.size, abi.ptr(b), abi.ptr(s),
                             abi.ptr(y), b.size, abi.ptr(out))
    if raise_errors or not (out["status"] != 0).any():
        check(rc)
    return out


def update_structural(params, cfg: LearnerConfig, b, s, y):
    """One learner: returns (accepted, params_after, counters)."""
    prob = problem_record(params, cfg, 0, len(b)).reshape(1)
    r = refit_batch(STRUCTURAL, prob, b, s, y)[0]
    return bool(r["updated"]), list(r["params"]), dict(zip(COUNTERS, r["counters"].tolist()))


def update_linear(params, cfg: LearnerConfig, b, s, y):
    prob = problem_record(params, cfg, 0, len(b)).reshape(1)
    r = refit_batch(LINEAR, prob, b, s, y)[0]
    return bool(r["updated"]), list(r["params"]), dict(zip(COUNTERS, r["counters"].tolist()))
