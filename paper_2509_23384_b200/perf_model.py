"""Perf-model API (mirror of proj/include/servesim/perf_model.h) on K1.

``throughput`` / ``predict_latency`` keep the reference signatures (a
PerfParams-like object or 8-sequence, and a (b, s) shape); ``eval_host`` /
``eval_device`` are the batched forms. Every call runs the sm_100a
perf_eval_kernel; invalid shapes or params raise ValueError like the
reference's std::invalid_argument (perf_model.cpp:22-29).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import astuple, dataclass

from ._lib import NX_DETERMINISTIC_FP64, NX_FAST_FP32, check, lib

FIELDS = ("tau0", "w0", "ws", "tauB", "tauS", "p_max", "kB", "kS")


@dataclass
class PerfParams:  # perf_model.h:14-27 (field order is the C layout)
    tau0: float = 0.0
    w0: float = 0.0
    ws: float = 1.0
    tauB: float = 0.0
    tauS: float = 0.0
    p_max: float = 1.0
    kB: float = 1.0
    kS: float = 1.0

    def valid(self) -> bool:
        return (self.p_max > 0 and self.kB > 0 and self.kS > 0 and self.tau0 >= 0 and
                self.tauB >= 0 and self.tauS >= 0 and self.ws > 0 and self.w0 >= 0)


PROFILES = {  # ground-truth tiers, engine.cpp:34-59
    "fast": PerfParams(4.0, 0.0, 1.0, 0.08, 0.0004, 20.0, 4.0, 0.05),
    "medium": PerfParams(5.0, 0.0, 1.0, 0.12, 0.0008, 10.0, 4.0, 0.05),
    "slow": PerfParams(6.0, 0.0, 1.0, 0.18, 0.0016, 5.0, 4.0, 0.05),
}
DEFAULT_PRIORS = PerfParams(5.0, 0.0, 1.0, 0.1, 0.001, 20.0, 0.1, 0.02)  # learner.cpp:117-128


def _row(p) -> list:
    if isinstance(p, PerfParams):
        return list(astuple(p))
    return [float(x) for x in p]


def eval_host(params_rows, idx, b, s, mode: int = NX_DETERMINISTIC_FP64, want_thr: bool = True):
    """Batched K1 on host arrays (copies in/out included). Returns (T, thr)."""
    import numpy as np
    P = np.ascontiguousarray(np.asarray([_row(p) for p in params_rows], dtype=np.float64))
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    n = idx.size
    T = np.empty(n, dtype=np.float64)
    thr = np.empty(n, dtype=np.float64) if want_thr else None
    check(lib().nx_perf_eval_host(P.ctypes.data, P.shape[0], idx.ctypes.data, b.ctypes.data,
                                  s.ctypes.data, T.ctypes.data,
                                  thr.ctypes.data if want_thr else None, n, mode))
    return T, thr


def eval_device(params, idx, b, s, out_T, out_thr=None, mode: int = NX_DETERMINISTIC_FP64,
                stream=None):
    """Batched K1 on torch CUDA tensors (float64 [n_params, 8]; int32 idx/b/s;
    float64 outputs), enqueued on `stream` (torch.cuda.Stream or None)."""
    sh = stream.cuda_stream if stream is not None else 0
    check(lib().nx_perf_eval_dev(params.data_ptr(), params.shape[0], idx.data_ptr(), b.data_ptr(),
                                 s.data_ptr(), out_T.data_ptr(),
                                 out_thr.data_ptr() if out_thr is not None else None,
                                 idx.numel(), mode, C.c_void_p(sh)))


def eval_device_async(params, idx, b, s, out_T, status, out_thr=None,
                      mode: int = NX_DETERMINISTIC_FP64, stream=None):
    """Stream-ordered K1 without host sync; `status` is an int32 CUDA tensor
    of one element the caller zeroes (nonzero afterwards = invalid input)."""
    sh = stream.cuda_stream if stream is not None else 0
    check(lib().nx_perf_eval_async(params.data_ptr(), params.shape[0], idx.data_ptr(),
                                   b.data_ptr(), s.data_ptr(), out_T.data_ptr(),
                                   out_thr.data_ptr() if out_thr is not None else None,
                                   idx.numel(), mode, status.data_ptr(), C.c_void_p(sh)))


def throughput(params, shape) -> float:
    """servesim::throughput(params, {b, s})."""
    b, s = shape
    _, thr = eval_host([params], [0], [b], [s])
    return float(thr[0])


def predict_latency(params, shape) -> float:
    """servesim::predict_latency(params, {b, s})."""
    b, s = shape
    T, _ = eval_host([params], [0], [b], [s], want_thr=False)
    return float(T[0])


def profile_table(device):
    import torch
    rows = [_row(PROFILES[k]) for k in ("fast", "medium", "slow")] + [_row(DEFAULT_PRIORS)]
    return torch.tensor(rows, dtype=torch.float64, device=device)


__all__ = ["PerfParams", "PROFILES", "DEFAULT_PRIORS", "eval_host", "eval_device", "throughput",
           "predict_latency", "NX_DETERMINISTIC_FP64", "NX_FAST_FP32"]
