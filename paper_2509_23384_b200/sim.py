"""Reference-facing simulation API (mirror of proj/include/servesim/sim.h).

``run_simulation``, ``sweep`` and the batched ``run_replicas`` take RunConfig
JSON documents in the reference's schema and return results shaped like
servesim::RunResult / SweepResult. All replicas of a call run in ONE launch of
the device lockstep kernel (one warp per replica); the host only parses
configs, synthesises workloads with the reference's generator semantics and
formats summaries.
"""
from __future__ import annotations

import copy
import ctypes as C
import json
import os
from dataclasses import dataclass, field

from . import _lib
from ._lib import RequestRecord, ReplicaSummary, check, lib


@dataclass
class RunResult:  # servesim::RunResult (sim.h:62-73)
    arrived: int
    completed: int
    rejected: int
    unfinished: int
    arrival_hash: int
    event_hash: int
    decisions: int
    events: int
    summary_json: str
    records: list = field(default_factory=list)
    learners: list = field(default_factory=list)   # (params8, samples, counters7) per engine
    learner_history: list = field(default_factory=list)  # LearnerSnapshot rows (sim.h:62-67)

    @property
    def summary(self) -> dict:
        return json.loads(self.summary_json)


def _texts(cfgs):
    return [c if isinstance(c, str) else json.dumps(c) for c in cfgs]


class Batch:
    """One device batch of replicas (an nx_sim handle)."""

    def __init__(self, cfgs, device: int = 0, host_threads: int | None = None):
        texts = _texts(cfgs)
        arr = (C.c_char_p * len(texts))(*[t.encode() for t in texts])
        h = C.c_void_p()
        threads = host_threads or max(1, os.cpu_count() or 1)
        check(lib().nx_sim_create_json(arr, len(texts), device, threads, C.byref(h)))
        self.h = h
        self.n = len(texts)

    def rebuild_workloads(self, host_threads: int | None = None):
        """Regenerate every replica's workload on the host (same results)."""
        check(lib().nx_sim_rebuild_workloads(self.h, host_threads or max(1, os.cpu_count() or 1)))

    def upload(self):
        check(lib().nx_sim_upload(self.h))

    def launch(self):
        check(lib().nx_sim_launch(self.h))

    def download(self):
        check(lib().nx_sim_download(self.h))

    def synchronize(self):
        check(lib().nx_sim_synchronize(self.h))

    def run(self):
        check(lib().nx_sim_run(self.h))
        return self

    def kernel_ms(self) -> float:
        v = C.c_float()
        check(lib().nx_sim_last_kernel_ms(self.h, C.byref(v)))
        return v.value

    def io_bytes(self):
        a, b = C.c_int64(), C.c_int64()
        check(lib().nx_sim_io_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def summaries(self):
        out = (ReplicaSummary * self.n)()
        check(lib().nx_sim_summaries(self.h, out))
        return list(out)

    def metrics(self, r: int) -> dict:
        """servesim::MetricsSummary of replica r, computed on the device (K7)."""
        m = _lib.ReplicaMetrics()
        check(lib().nx_sim_metrics(self.h, r, C.byref(m)))
        return {k: getattr(m, k) for k, _ in m._fields_}

    def summary_json(self, r: int) -> str:
        n = C.c_int64()
        check(lib().nx_sim_summary_json(self.h, r, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().nx_sim_summary_json(self.h, r, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def records(self, r: int):
        n = C.c_int64()
        check(lib().nx_sim_records(self.h, r, None, 0, C.byref(n)))
        arr = (RequestRecord * max(1, n.value))()
        check(lib().nx_sim_records(self.h, r, arr, n.value, C.byref(n)))
        return list(arr)[: n.value]

    def work(self, r: int):
        out = (C.c_int64 * 6)()
        check(lib().nx_sim_work(self.h, r, out))
        return list(out)

    def phase_cycles(self, r: int):
        out = (C.c_int64 * 16)()
        check(lib().nx_sim_phase_cycles(self.h, r, out))
        return list(out)

    def timeline(self, r: int):
        """(begin_ns, end_ns) of replica r on the device's %globaltimer."""
        out = (C.c_int64 * 2)()
        check(lib().nx_sim_timeline(self.h, r, out))
        return out[0], out[1]

    def summaries_nbytes(self) -> int:
        ptr, n = C.c_void_p(), C.c_int64()
        check(lib().nx_sim_summaries_dev(self.h, C.byref(ptr), C.byref(n)))
        return n.value

    def gather_summaries(self, comm, recv_ptr: int):
        """K6: ncclAllGather of every rank's summaries into recv_ptr (device;
        world x summaries_nbytes), on this batch's stream."""
        check(lib().nx_sim_gather_summaries(self.h, comm.handle, C.c_void_p(recv_ptr)))

    def copy_summaries(self, dst_ptr: int):
        check(lib().nx_sim_copy_summaries(self.h, C.c_void_p(dst_ptr)))

    def learner(self, r: int, e: int):
        p = (C.c_double * 8)()
        s = C.c_int64()
        cnt = (C.c_int64 * 7)()
        check(lib().nx_sim_learner(self.h, r, e, p, C.byref(s), cnt))
        return list(p), s.value, list(cnt)

    def _rows(self, fn, row, r):
        n = C.c_int64()
        check(getattr(lib(), fn)(self.h, r, None, 0, C.byref(n)))
        arr = (row * max(1, n.value))()
        check(getattr(lib(), fn)(self.h, r, arr, n.value, C.byref(n)))
        return list(arr)[: n.value]

    def plan_log(self, r: int):
        """plans_jsonl rows (sim.cpp:149-158) written by the device."""
        return [{"sim_time": x.sim_time_ms, "engine_id": x.engine_id, "b": x.b, "s": x.s,
                 "predicted_ms": x.predicted_ms, "target_ms": x.target_ms}
                for x in self._rows("nx_sim_plan_log", _lib.PlanLogRow, r)]

    def route_log(self, r: int):
        """routing_jsonl rows (sim.cpp:176-186) written by the device."""
        return [{"sim_time": x.sim_time_ms, "request_id": x.request_id, "chosen_engine": x.chosen_engine,
                 "s_latency": x.s_latency, "s_load": x.s_load, "s_capacity": x.s_capacity,
                 "s_affinity": x.s_affinity, "score": x.score}
                for x in self._rows("nx_sim_route_log", _lib.RouteLogRow, r)]

    def learner_history(self, r: int):
        """RunResult::learner_history (sim.cpp:322-327): (engine_id, sim_time_ms,
        samples_seen, params[8]) after every learner update event."""
        return [(x.engine_id, x.sim_time_ms, x.samples_seen, list(x.params))
                for x in self._rows("nx_sim_learner_history", _lib.LearnerSnapshot, r)]

    def write_outputs(self, r: int):
        """Simulation::write_outputs (sim.cpp:393-413) into the config's output.dir."""
        check(lib().nx_sim_write_outputs(self.h, r))

    def error(self, r: int) -> str:
        """The reference's exception text for a failed replica ('' if it ran)."""
        buf = C.create_string_buffer(512)
        lib().nx_sim_error(self.h, r, buf, 512)
        return buf.value.decode()

    def result(self, r: int, with_records: bool = True, n_engines: int | None = None) -> RunResult:
        s = self.summaries()[r]
        if s.status != 0:
            _raise_status(s, self.error(r))
        sj = self.summary_json(r)
        ne = n_engines if n_engines is not None else len(json.loads(sj)["learners"])
        return RunResult(s.arrived, s.completed, s.rejected, s.unfinished, s.arrival_hash,
                         s.event_hash, s.decisions, s.events, sj,
                         self.records(r) if with_records else [],
                         [self.learner(r, e) for e in range(ne)])

    def close(self):
        if getattr(self, "h", None):
            lib().nx_sim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _raise_status(s, msg: str = ""):
    msg = msg or f"device replica failed at site {s.err_site}"
    if s.status == _lib.NX_EINVAL:
        raise ValueError(msg)
    if s.status == _lib.NX_ELOGIC:
        raise _lib.LogicError(msg)
    raise RuntimeError(msg)


def run_replicas(cfgs, device: int = 0, with_records: bool = False):
    b = Batch(cfgs, device).run()
    try:
        return [b.result(r, with_records) for r in range(b.n)]
    finally:
        b.close()


def run_simulation(cfg, device: int = 0) -> RunResult:
    """servesim::run_simulation (sim.cpp:596-599) on the device; writes the
    output files when the config names an output.dir (sim.cpp:345)."""
    b = Batch([cfg], device).run()
    try:
        res = b.result(0, True)
        res.learner_history = b.learner_history(0)
        b.write_outputs(0)
        return res
    finally:
        b.close()


def sweep(base: dict, axis: str, values, device: int = 0):
    """servesim::sweep (sim.cpp:608-642): every value becomes one replica of a
    single device batch instead of a sequential loop. Per-value failures are
    reported per row, like the reference."""
    if axis not in ("rate", "policy", "budget"):
        raise RuntimeError(f"unknown sweep axis: {axis}")
    rows = [{"value": str(v), "ok": False, "error": ""} for v in values]
    cfgs, where = [], []
    for i, v in enumerate(values):
        try:
            c = copy.deepcopy(base)
            c.setdefault("output", {})["dir"] = ""
            if axis == "rate":
                c.setdefault("workload", {})["mode"] = "qps"
                c["workload"]["rate"] = float(v)
            elif axis == "policy":
                for e in c["engines"]:
                    e["scheduler_policy"] = v
            else:
                for e in c["engines"]:
                    e["static_budget"] = int(v)
            workload_info(c)  # parse + validate + build the workload (host only)
        except Exception as exc:  # noqa: BLE001 — the row records it (sim.cpp:608-642)
            rows[i]["error"] = str(exc)
            continue
        cfgs.append(c)
        where.append(i)
    if not cfgs:
        return {"axis": axis, "rows": rows}
    b = Batch(cfgs, device).run()
    try:
        sums = b.summaries()
        for k, i in enumerate(where):
            if sums[k].status != 0:
                rows[i]["error"] = b.error(k)
            else:
                rows[i] = {"value": rows[i]["value"], "ok": True, "result": b.result(k, False)}
    finally:
        b.close()
    return {"axis": axis, "rows": rows}


def workload_info(cfg):
    """Host-only: (arrival_hash, n_requests, n_sessions) of a RunConfig."""
    h, n, ns = C.c_uint64(), C.c_int64(), C.c_int64()
    text = cfg if isinstance(cfg, str) else json.dumps(cfg)
    check(lib().nx_workload_info(text.encode(), C.byref(h), C.byref(n), C.byref(ns)))
    return h.value, n.value, ns.value


def synth_generate(scenario: str, n: int, seed: int):
    """workload.cpp:137-166 semantics -> (prompts, outputs, session_ids)."""
    P = (C.c_int64 * n)()
    O = (C.c_int64 * n)()
    S = C.create_string_buffer(16 * n)
    check(lib().nx_synth_generate(scenario.encode(), n, seed, P, O, S))
    raw = S.raw
    sess = [raw[16 * i:16 * i + 16].split(b"\0", 1)[0].decode() for i in range(n)]
    return list(P), list(O), sess
