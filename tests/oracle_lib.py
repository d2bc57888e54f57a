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


class Port(_Lib):
    prefix = "port_"

    def __init__(self):
        super().__init__(PORT_SO)


def ref_available() -> bool:
    return REF_SO.exists()
