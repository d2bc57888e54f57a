"""TEST INFRASTRUCTURE — ctypes access to the two CPU checkers.

* ``Ref``  : oracle/_ref/libservesim_ref.so — the unmodified reference core
             (/root/reference/proj/src) + oracle/ref_driver.cpp.
* ``Port`` : oracle/_port/libnx_oracle.so — the flat CPU restatement
             (oracle/port/*.cpp).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / reference
arm) may use this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libservesim_ref.so"
PORT_SO = ROOT / "oracle" / "_port" / "libnx_oracle.so"

_P = C.POINTER


class _Lib:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(str(path))
        p = self.prefix
        L = self.lib
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "run_json").argtypes = [C.c_char_p, C.c_int, _P(C.c_void_p)]
        getattr(L, p + "run_batch").argtypes = [
            _P(C.c_char_p), C.c_int, C.c_int, _P(C.c_int64), _P(C.c_uint64), _P(C.c_double)]
        getattr(L, p + "free").argtypes = [C.c_void_p]
        getattr(L, p + "perf_eval").argtypes = [
            _P(C.c_double), _P(C.c_int64), _P(C.c_int64), C.c_int64, _P(C.c_double), _P(C.c_double)]

    def err(self) -> str:
        return getattr(self.lib, self.prefix + "last_error")().decode()

    def run(self, cfg: dict | str, records: bool = False) -> dict:
        text = cfg if isinstance(cfg, str) else json.dumps(cfg)
        out = C.c_void_p()
        rc = getattr(self.lib, self.prefix + "run_json")(text.encode(), int(records), C.byref(out))
        if rc != 0:
            raise RuntimeError(f"{self.prefix}run_json rc={rc}: {self.err()}")
        s = C.cast(out, C.c_char_p).value.decode()
        getattr(self.lib, self.prefix + "free")(out)
        return json.loads(s)

    def run_batch(self, cfgs: list, threads: int):
        n = len(cfgs)
        texts = (C.c_char_p * n)(*[(c if isinstance(c, str) else json.dumps(c)).encode() for c in cfgs])
        dec = (C.c_int64 * n)()
        eh = (C.c_uint64 * n)()
        wall = C.c_double()
        rc = getattr(self.lib, self.prefix + "run_batch")(texts, n, threads, dec, eh, C.byref(wall))
        if rc != 0:
            raise RuntimeError(f"{self.prefix}run_batch rc={rc}: {self.err()}")
        return list(dec), list(eh), wall.value

    def perf_eval(self, params8, b, s):
        import numpy as np
        b = np.ascontiguousarray(b, dtype=np.int64)
        s = np.ascontiguousarray(s, dtype=np.int64)
        p = (C.c_double * 8)(*params8)
        T = np.empty(len(b))
        thr = np.empty(len(b))
        rc = getattr(self.lib, self.prefix + "perf_eval")(
            p, b.ctypes.data_as(_P(C.c_int64)), s.ctypes.data_as(_P(C.c_int64)), len(b),
            T.ctypes.data_as(_P(C.c_double)), thr.ctypes.data_as(_P(C.c_double)))
        if rc != 0:
            raise ValueError(self.err())
        return T, thr


class Ref(_Lib):
    prefix = "ref_"

    def __init__(self):
        super().__init__(REF_SO)
        L = self.lib
        V = C.c_void_p
        L.ref_schedule_step.argtypes = [V, V, C.c_int64, C.c_int64, C.c_double, C.c_double, V, V,
                                        C.c_int64, C.c_int64, C.c_int, C.c_double, C.c_double,
                                        V, V, V, V, V, V]
        L.ref_schedule_baseline.argtypes = [C.c_int, V, V, C.c_int64, C.c_int64, V, C.c_int64,
                                            C.c_int64, C.c_int64, C.c_int, V, V, V, V, V]
        L.ref_route_group.argtypes = [C.c_int, V, C.c_double, C.c_double, C.c_uint64, C.c_int, V, V,
                                      V, V, V, C.c_int, V, V, V, C.c_int, V, V, V, V, V, V, V, V, V]
        L.ref_learner_linear.argtypes = [V, C.c_int64, C.c_int64, V, V, V, C.c_int64, V, V, V]
        L.ref_learner_structural2.argtypes = [V, C.c_int64, C.c_int64, C.c_int64, V, V, V,
                                              C.c_int64, V, V, V]

    # ---- per-operator oracles (unmodified servesim:: calls, ref_driver.cpp) ----
    def schedule_step(self, n_run, wait_prompt, wait_prefilled, ttft, tpot, tm4, params8,
                      m_max, q_max, n_iters, eps, q_ref):
        import numpy as np
        wp = np.ascontiguousarray(wait_prompt, dtype=np.int64)
        wf = np.ascontiguousarray(wait_prefilled, dtype=np.int64)
        tm = np.ascontiguousarray(tm4, dtype=np.float64)
        pp = np.ascontiguousarray(params8, dtype=np.float64)
        n_alloc = n_run + wp.size + 1
        bs = np.zeros(2, dtype=np.int64)
        pt = np.zeros(2, dtype=np.float64)
        ov = np.zeros(1, dtype=np.int32)
        aid = np.zeros(n_alloc, dtype=np.int64)
        atok = np.zeros(n_alloc, dtype=np.int64)
        apf = np.zeros(n_alloc, dtype=np.int32)
        rc = self.lib.ref_schedule_step(wp.ctypes.data, wf.ctypes.data, wp.size, n_run, ttft, tpot,
                                        tm.ctypes.data, pp.ctypes.data, m_max, q_max, n_iters, eps,
                                        q_ref, bs.ctypes.data, pt.ctypes.data, ov.ctypes.data,
                                        aid.ctypes.data, atok.ctypes.data, apf.ctypes.data)
        if rc != 0:
            return {"status": rc}
        b = int(bs[0])
        return {"status": 0, "b": b, "s": int(bs[1]), "predicted": float(pt[0]),
                "target": float(pt[1]), "overload": int(ov[0]),
                "alloc": [(int(aid[i]), int(atok[i]), int(apf[i])) for i in range(b)]}

    def schedule_baseline(self, policy, n_run, wait_prompt, wait_prefilled, params8, m_max, q_max,
                          static_budget, engine_id=0):
        import numpy as np
        wp = np.ascontiguousarray(wait_prompt, dtype=np.int64)
        wf = np.ascontiguousarray(wait_prefilled, dtype=np.int64)
        pp = np.ascontiguousarray(params8, dtype=np.float64)
        n_alloc = n_run + wp.size + 1
        bs = np.zeros(2, dtype=np.int64)
        pr = np.zeros(1, dtype=np.float64)
        aid = np.zeros(n_alloc, dtype=np.int64)
        atok = np.zeros(n_alloc, dtype=np.int64)
        apf = np.zeros(n_alloc, dtype=np.int32)
        rc = self.lib.ref_schedule_baseline(policy, wp.ctypes.data, wf.ctypes.data, wp.size, n_run,
                                            pp.ctypes.data, m_max, q_max, static_budget, engine_id,
                                            bs.ctypes.data, pr.ctypes.data, aid.ctypes.data,
                                            atok.ctypes.data, apf.ctypes.data)
        if rc != 0:
            return {"status": rc}
        b = int(bs[0])
        return {"status": 0, "b": b, "s": int(bs[1]), "predicted": float(pr[0]),
                "alloc": [(int(aid[i]), int(atok[i]), int(apf[i])) for i in range(b)]}

    def route_group(self, policy, cfg9, ttft, tpot, seed, ids, static_w, states5, qlen, has_rep,
                    comp_engine, comp_session, comp_decode, req_prompt, req_session, req_now):
        import numpy as np
        f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
        cfg9, static_w, states5, req_now = f64(cfg9), f64(static_w), f64(states5), f64(req_now)
        ids, has_rep, comp_engine, comp_session, req_session = (i32(ids), i32(has_rep), i32(comp_engine),
                                                                 i32(comp_session), i32(req_session))
        qlen, comp_decode, req_prompt = i64(qlen), i64(comp_decode), i64(req_prompt)
        n, m = ids.size, req_prompt.size
        eng = np.zeros(m, dtype=np.int32)
        score = np.zeros(m)
        fac = np.zeros(4 * m)
        deg = np.zeros(m, dtype=np.int32)
        st5 = np.zeros(5 * n)
        oq = np.zeros(n, dtype=np.int64)
        d = lambda a: a.ctypes.data
        rc = self.lib.ref_route_group(policy, d(cfg9), ttft, tpot, seed, n, d(ids), d(static_w),
                                      d(states5), d(qlen), d(has_rep), comp_engine.size,
                                      d(comp_engine), d(comp_session), d(comp_decode), m,
                                      d(req_prompt), d(req_session), d(req_now), d(eng), d(score),
                                      d(fac), d(deg), d(st5), d(oq))
        if rc != 0:
            return {"status": rc}
        return {"status": 0, "engine": eng, "score": score, "factors": fac.reshape(m, 4),
                "degraded": deg, "states5": st5.reshape(n, 5), "qlen": oq}

    def learner_refit(self, kind, priors8, long_w, short_w, min_s, b, s, y):
        import numpy as np
        b = np.ascontiguousarray(b, dtype=np.int64)
        s = np.ascontiguousarray(s, dtype=np.int64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        pp = np.ascontiguousarray(priors8, dtype=np.float64)
        out = np.zeros(8)
        acc = np.zeros(1, dtype=np.int32)
        cnt = np.zeros(7, dtype=np.int64)
        if kind == 0:
            rc = self.lib.ref_learner_linear(pp.ctypes.data, long_w, short_w, b.ctypes.data,
                                             s.ctypes.data, y.ctypes.data, b.size, out.ctypes.data,
                                             acc.ctypes.data, cnt.ctypes.data)
        else:
            rc = self.lib.ref_learner_structural2(pp.ctypes.data, long_w, short_w, min_s,
                                                  b.ctypes.data, s.ctypes.data, y.ctypes.data,
                                                  b.size, out.ctypes.data, acc.ctypes.data,
                                                  cnt.ctypes.data)
        if rc != 0:
            return {"status": rc}
        return {"status": 0, "params": out, "updated": int(acc[0]), "counters": cnt}


class Port(_Lib):
    prefix = "port_"

    def __init__(self):
        super().__init__(PORT_SO)


def ref_available() -> bool:
    return REF_SO.exists()
