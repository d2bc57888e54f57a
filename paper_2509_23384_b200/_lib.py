"""ctypes binding of include/nx_sched.h (the product's C-ABI).

The shared library is built in-tree (paper_2509_23384_b200/_nxsched.so) by
``__graft_entry__.build()``. There is no fallback: if it is missing, or no
CUDA device is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

SO_PATH = Path(__file__).resolve().parent / os.environ.get("NX_SO", "_nxsched.so")

NX_OK, NX_EINVAL, NX_ERUNTIME, NX_ELOGIC, NX_ECUDA = 0, 1, 2, 3, 4
NX_DETERMINISTIC_FP64, NX_FAST_FP32 = 0, 1


class CudaError(RuntimeError):
    """A CUDA call failed (no device, out of memory, launch failure)."""


class LogicError(RuntimeError):
    """Mirror of std::logic_error (internal invariant violated)."""


class ReplicaSummary(C.Structure):
    _fields_ = [("arrived", C.c_int64), ("completed", C.c_int64), ("rejected", C.c_int64),
                ("unfinished", C.c_int64), ("events", C.c_int64), ("decisions", C.c_int64),
                ("arrival_hash", C.c_uint64), ("event_hash", C.c_uint64),
                ("status", C.c_int32), ("err_site", C.c_int32)]


class ReplicaMetrics(C.Structure):  # nx_replica_metrics (servesim::MetricsSummary)
    _fields_ = [("completed", C.c_int64), ("p50_e2e_ms", C.c_double), ("p90_e2e_ms", C.c_double),
                ("p50_ttft_ms", C.c_double), ("p50_tpot_ms", C.c_double), ("mean_ttft_ms", C.c_double),
                ("mean_tpot_ms", C.c_double), ("slo_attainment_pct", C.c_double)]


class RequestRecord(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("arrival_ms", C.c_double),
                ("first_token_ms", C.c_double), ("completed_ms", C.c_double),
                ("prompt_tokens", C.c_int64), ("output_tokens", C.c_int64),
                ("engine_id", C.c_int32), ("pad_", C.c_int32)]


class PlanLogRow(C.Structure):
    _fields_ = [("sim_time_ms", C.c_double), ("engine_id", C.c_int32), ("pad_", C.c_int32),
                ("b", C.c_int64), ("s", C.c_int64), ("predicted_ms", C.c_double),
                ("target_ms", C.c_double)]


class RouteLogRow(C.Structure):
    _fields_ = [("sim_time_ms", C.c_double), ("request_id", C.c_int64), ("chosen_engine", C.c_int32),
                ("pad_", C.c_int32), ("s_latency", C.c_double), ("s_load", C.c_double),
                ("s_capacity", C.c_double), ("s_affinity", C.c_double), ("score", C.c_double)]


class LearnerSnapshot(C.Structure):
    _fields_ = [("engine_id", C.c_int32), ("pad_", C.c_int32), ("sim_time_ms", C.c_double),
                ("samples_seen", C.c_int64), ("params", C.c_double * 8)]


_lib = None
_P = C.POINTER


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not SO_PATH.exists():
        raise FileNotFoundError(
            f"{SO_PATH} is not built — run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(str(SO_PATH))
    L.nx_last_error.restype = C.c_char_p
    L.nx_device_count.restype = C.c_int
    L.nx_sim_create_json.argtypes = [_P(C.c_char_p), C.c_int32, C.c_int32, C.c_int32, _P(C.c_void_p)]
    for fn in ("nx_sim_upload", "nx_sim_launch", "nx_sim_download", "nx_sim_synchronize",
               "nx_sim_run", "nx_sim_replica_count"):
        getattr(L, fn).argtypes = [C.c_void_p]
    L.nx_sim_last_kernel_ms.argtypes = [C.c_void_p, _P(C.c_float)]
    L.nx_sim_io_bytes.argtypes = [C.c_void_p, _P(C.c_int64), _P(C.c_int64)]
    L.nx_sim_summaries.argtypes = [C.c_void_p, _P(ReplicaSummary)]
    L.nx_sim_error.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int64]
    L.nx_sim_rebuild_workloads.argtypes = [C.c_void_p, C.c_int32]
    L.nx_sim_summary_json.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int64, _P(C.c_int64)]
    L.nx_sim_metrics.argtypes = [C.c_void_p, C.c_int32, _P(ReplicaMetrics)]
    L.nx_sim_records.argtypes = [C.c_void_p, C.c_int32, _P(RequestRecord), C.c_int64, _P(C.c_int64)]
    L.nx_sim_learner.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _P(C.c_double), _P(C.c_int64),
                                 _P(C.c_int64)]
    L.nx_sim_destroy.argtypes = [C.c_void_p]
    L.nx_sim_destroy.restype = None
    L.nx_sim_work.argtypes = [C.c_void_p, C.c_int32, _P(C.c_int64)]
    L.nx_sim_phase_cycles.argtypes = [C.c_void_p, C.c_int32, _P(C.c_int64)]
    L.nx_sim_timeline.argtypes = [C.c_void_p, C.c_int32, _P(C.c_int64)]
    L.nx_sim_copy_summaries.argtypes = [C.c_void_p, C.c_void_p]
    L.nx_sim_summaries_dev.argtypes = [C.c_void_p, _P(C.c_void_p), _P(C.c_int64)]
    L.nx_perf_eval_dev.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]
    L.nx_perf_eval_async.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                     C.c_void_p]
    L.nx_perf_eval_host.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_int64, C.c_int32]
    L.nx_workload_info.argtypes = [C.c_char_p, _P(C.c_uint64), _P(C.c_int64), _P(C.c_int64)]
    L.nx_synth_generate.argtypes = [C.c_char_p, C.c_int64, C.c_uint64, _P(C.c_int64),
                                    _P(C.c_int64), C.c_char_p]
    V = C.c_void_p
    for fn, row in (("nx_sim_plan_log", PlanLogRow), ("nx_sim_route_log", RouteLogRow),
                    ("nx_sim_learner_history", LearnerSnapshot)):
        getattr(L, fn).argtypes = [C.c_void_p, C.c_int32, _P(row), C.c_int64, _P(C.c_int64)]
    L.nx_sim_write_outputs.argtypes = [C.c_void_p, C.c_int32]
    L.nx_nccl_unique_id.argtypes = [C.c_char_p]
    L.nx_nccl_comm_init.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _P(C.c_void_p)]
    L.nx_nccl_comm_destroy.argtypes = [C.c_void_p]
    L.nx_sim_gather_summaries.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    L.nx_rng_state.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64, _P(C.c_uint64)]
    L.nx_abi_sizes.argtypes = [_P(C.c_int64), C.c_int32]
    L.nx_lens_schedule_dev.argtypes = [V, C.c_int32, V, C.c_int64, V, V, V]
    L.nx_lens_schedule_host.argtypes = [V, C.c_int32, V, C.c_int64, V, V]
    L.nx_lens_schedule_mode_dev.argtypes = [V, C.c_int32, V, C.c_int64, V, V, C.c_int32, V]
    L.nx_lens_schedule_mode_host.argtypes = [V, C.c_int32, V, C.c_int64, V, V, C.c_int32]
    L.nx_baseline_schedule_host.argtypes = [V, C.c_int32, V, C.c_int64, V]
    L.nx_prism_route_dev.argtypes = [V, C.c_int32, V, V, V, V, V, V]
    L.nx_prism_route_host.argtypes = [V, C.c_int32, V, C.c_int64, V, C.c_int64, V, C.c_int64, V, V]
    L.nx_prism_route_mode_dev.argtypes = [V, C.c_int32, V, V, V, V, V, C.c_int32, V]
    L.nx_prism_route_mode_host.argtypes = [V, C.c_int32, V, C.c_int64, V, C.c_int64, V, C.c_int64, V, V, C.c_int32]
    L.nx_refit_dev.argtypes = [C.c_int32, V, C.c_int32, V, V, V, C.c_int64, V, V]
    L.nx_refit_host.argtypes = [C.c_int32, V, C.c_int32, V, V, V, C.c_int64, V]
    _lib = L
    return L


def check(rc: int) -> None:
    """Map an nx status to the Python analogue of the reference exception."""
    if rc == NX_OK:
        return
    msg = lib().nx_last_error().decode(errors="replace")
    if rc == NX_EINVAL:
        raise ValueError(msg)          # std::invalid_argument
    if rc == NX_ELOGIC:
        raise LogicError(msg)          # std::logic_error
    if rc == NX_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)            # std::runtime_error
