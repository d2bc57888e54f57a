"""Deterministic per-operator parity cases for the batched K2/K3/K4 entry
points (nx_lens_schedule, nx_prism_route, nx_refit).

The scenarios follow the reference's own unit tests — tests/test_lens.cpp
(empty queues :231-236, single decode :238-246, full-scan sweep :248-293,
overload :319-330, feasibility invariants :332-372), tests/test_router.cpp
and tests/test_learner.cpp — widened with random shapes (long queues,
q_max spans beyond the shared-memory stage, stale / missing reports, every
routing policy, saturated and degenerate learner windows).
"""
from __future__ import annotations

import math

import numpy as np

FAST = [4.0, 0.0, 1.0, 0.08, 0.0004, 20.0, 4.0, 0.05]   # engine.cpp:34-59 (PerfParams order)
MEDIUM = [5.0, 0.0, 1.0, 0.12, 0.0008, 10.0, 4.0, 0.05]
SLOW = [6.0, 0.0, 1.0, 0.18, 0.0016, 5.0, 4.0, 0.05]
PRIORS = [5.0, 0.0, 1.0, 0.1, 0.001, 20.0, 0.1, 0.02]   # learner.cpp:117-128
TM_BASE = [100.0, 10.0, 200.0, 1.0]                     # test_lens.cpp:16-24


def _lens(n_run, rem, prefilled=None, ttft=40.0, tpot=12.0, tm=TM_BASE, params=FAST,
          m_max=8192, q_max=256, n_iters=10, eps=0.05, q_ref=16.0):
    rem = [int(x) for x in rem]
    pre = [0] * len(rem) if prefilled is None else [int(x) for x in prefilled]
    return {"n_run": int(n_run), "prompt": [r + p for r, p in zip(rem, pre)], "prefilled": pre,
            "ttft": float(ttft), "tpot": float(tpot), "tm": [float(x) for x in tm],
            "params": [float(x) for x in params], "m_max": int(m_max), "q_max": int(q_max),
            "n_iters": int(n_iters), "eps": float(eps), "q_ref": float(q_ref)}


def _perturb(rng, base):
    p = list(base)
    p[0] = base[0] * rng.uniform(0.2, 3.0)                  # tau0
    p[3] = base[3] * rng.uniform(0.2, 3.0)                  # tauB
    p[4] = base[4] * rng.uniform(0.2, 3.0)                  # tauS
    p[5] = base[5] * rng.uniform(0.3, 3.0)                  # p_max
    p[6] = math.exp(rng.uniform(math.log(0.01), math.log(20.0)))   # kB
    p[7] = math.exp(rng.uniform(math.log(1e-4), math.log(0.5)))    # kS
    return p


def lens_cases():
    rng = np.random.default_rng(2509)
    out = []
    out.append(_lens(0, []))                                         # empty plan
    out.append(_lens(1, []))                                         # single decode
    out.append(_lens(6, [], q_max=4, m_max=8192))                    # overload
    out.append(_lens(300, [100, 200], q_max=256))                    # overload with waiters
    for _ in range(50):                                              # full-scan sweep trials
        out.append(_lens(4, rng.integers(1, 2001, 6), params=MEDIUM, eps=1e-12, n_iters=20))
    for _ in range(50):                                              # same, eager early exit
        out.append(_lens(4, rng.integers(1, 2001, 6), params=MEDIUM, eps=0.05, n_iters=20))
    for _ in range(200):                                             # feasibility invariants
        q = int(1 + rng.integers(0, 16))
        m = q + int(rng.integers(0, 4096))
        out.append(_lens(int(rng.integers(0, q + 1)), rng.integers(1, 3001, int(rng.integers(0, 8))),
                         params=SLOW, q_max=q, m_max=m))
    for _ in range(200):                                             # random long queues
        R = int(rng.integers(0, 257))
        W = int(rng.integers(0, 600))
        rem = np.exp(rng.uniform(0, math.log(30000), W)).astype(np.int64) + 1
        pre = rng.integers(0, 64, W)
        base = [FAST, MEDIUM, SLOW, PRIORS][int(rng.integers(0, 4))]
        tm = [rng.uniform(50, 8000), rng.uniform(0.5, 300), rng.uniform(1, 600), rng.uniform(0.5, 5)]
        out.append(_lens(R, rem, pre, ttft=rng.uniform(100, 5000), tpot=rng.uniform(5, 80), tm=tm,
                         params=_perturb(rng, base), m_max=int(rng.choice([2048, 8192, 16384])),
                         q_max=256, n_iters=int(rng.choice([6, 10, 14])),
                         eps=float(rng.choice([0.01, 0.05, 0.2])), q_ref=float(rng.choice([4, 16, 64]))))
    for _ in range(6):                                               # spans beyond 1024 waiters
        W = 1500
        out.append(_lens(int(rng.integers(0, 40)), rng.integers(1, 200, W), q_max=2048, m_max=65536,
                         params=_perturb(rng, FAST), ttft=3000.0, tpot=60.0))
    # invalid inputs -> std::invalid_argument
    out.append(_lens(2, [10], tpot=-1.0))                            # SLOSpec
    out.append(_lens(2, [10], eps=1.5))                              # SchedulerConfig
    out.append(_lens(2, [10], params=[1, 0, 1, 0, 0, 10, -1.0, 0.05]))   # PerfParams
    out.append(_lens(2, [10], tm=[100.0, -2.0, 200.0, 1.0]))         # TradeoffModel
    out.append(_lens(2, [10], ttft=1e9, tm=[10.0, 1.0, 0.5, 1.0], tpot=1e-300))  # tiny target
    return out


# ---- schedule_baseline (engine.cpp:61-108) ---------------------------------------
def _base(policy, n_run, rem, prefilled=None, params=FAST, m_max=8192, q_max=256, static_budget=2048,
          engine_id=0):
    rem = [int(x) for x in rem]
    pre = [0] * len(rem) if prefilled is None else [int(x) for x in prefilled]
    return {"policy": int(policy), "n_run": int(n_run), "prompt": [r + p for r, p in zip(rem, pre)],
            "prefilled": pre, "params": [float(x) for x in params], "m_max": int(m_max),
            "q_max": int(q_max), "static_budget": int(static_budget), "engine_id": int(engine_id)}


def baseline_cases():
    rng = np.random.default_rng(61108)
    out = []
    for pol in (1, 2):
        out.append(_base(pol, 0, []))                                # empty plan
        out.append(_base(pol, 5, []))                                # decodes only
        out.append(_base(pol, 5, [300, 400], q_max=64))              # test_engine.cpp:282-352 shapes
        out.append(_base(pol, 3, [1000], static_budget=512, q_max=64))
    out.append(_base(1, 0, [9000], m_max=8192, engine_id=7))         # first prompt > m_max: runtime_error
    out.append(_base(1, 2, [100, 9000, 5], m_max=8192))              # stops at the first misfit
    out.append(_base(1, 0, [10] * 40, q_max=16))                     # q_max cap
    out.append(_base(2, 300, [10], q_max=256))                       # |run| > q_max: invalid_argument
    out.append(_base(0, 1, [10]))                                    # lens policy: logic_error
    out.append(_base(2, 1, [10], params=[1, 0, 1, 0, 0, 10, -1.0, 0.05]))   # invalid params
    for _ in range(300):
        pol = int(rng.integers(1, 3))
        q = int(rng.integers(1, 300))
        m = q + int(rng.integers(0, 20000))
        R = int(rng.integers(0, q + 1))
        W = int(rng.integers(0, 400))
        rem = np.exp(rng.uniform(0, math.log(12000), W)).astype(np.int64) + 1
        pre = rng.integers(0, 64, W)
        base = [FAST, MEDIUM, SLOW, PRIORS][int(rng.integers(0, 4))]
        sb = int(rng.integers(1, m + 1))
        out.append(_base(pol, R, rem, pre, params=_perturb(rng, base), m_max=m, q_max=q,
                         static_budget=sb, engine_id=int(rng.integers(0, 16))))
    return out


# ---- K3 ------------------------------------------------------------------------
def _cfg9(rng, weights=None):
    w = weights if weights is not None else [float(rng.choice([0.0, 0.5, 1.0, 1.0, 2.0])) for _ in range(4)]
    return w + [float(rng.uniform(1.1, 3.0)), float(rng.uniform(0.0, 1.0)),
                float(rng.choice([0.0, 50.0, 400.0])), float(rng.uniform(5.0, 200.0)),
                float(rng.uniform(1.0, 4.0))]


def route_cases():
    rng = np.random.default_rng(4242)
    out = []
    for trial in range(160):
        policy = [0, 0, 0, 1, 2, 3, 5][trial % 7]
        n = int(rng.choice([1, 2, 4, 8, 8, 13, 32]))
        ids = [int(x) for x in rng.permutation(np.arange(100, 100 + 3 * n))[:n]]
        now0 = float(rng.uniform(0, 5000))
        has = [int(rng.random() < 0.85) for _ in range(n)]
        stale_all = trial % 11 == 5
        states = []
        for e in range(n):
            age = rng.uniform(2000, 9000) if stale_all or rng.random() < 0.2 else rng.uniform(0, 900)
            states.append([float(rng.uniform(0, 3000)) if rng.random() < 0.7 else 0.0,
                           float(rng.uniform(0, 50000)), float(rng.uniform(-1000, 200000)),
                           float(rng.uniform(1, 40)), now0 - age])
        qlen = [int(x) for x in rng.integers(0, 60, n)]
        static_w = [float(rng.choice([1.0, 0.5, 2.0, 3.0])) for _ in range(n)]
        n_sess = int(rng.integers(1, 40))
        n_comp = int(rng.integers(0, 30))
        comp_engine = [int(ids[int(rng.integers(0, n))]) if rng.random() < 0.9 else 999 for _ in range(n_comp)]
        comp_session = [int(x) for x in rng.integers(0, n_sess, n_comp)]
        comp_decode = [int(x) for x in rng.integers(0, 900, n_comp)]
        m = int(rng.integers(1, 64))
        req_prompt = [int(x) for x in rng.integers(1, 20000, m)]
        req_session = [int(x) for x in rng.integers(0, n_sess, m)]
        req_now = list(now0 + np.cumsum(rng.uniform(0, 50, m)))
        out.append({"policy": policy, "cfg9": _cfg9(rng), "ttft": float(rng.uniform(200, 4000)),
                    "tpot": 30.0, "seed": int(rng.integers(1, 2 ** 40)), "ids": ids,
                    "static_w": static_w, "states5": states, "qlen": qlen, "has_report": has,
                    "comp_engine": comp_engine, "comp_session": comp_session,
                    "comp_decode": comp_decode, "n_sessions": n_sess, "req_prompt": req_prompt,
                    "req_session": req_session, "req_now": req_now})
    return out


# ---- K4 ------------------------------------------------------------------------
def _predict(p, b, s):
    """predict_latency in float64 (sample synthesis only; any doubles will do)."""
    fb = min(-math.expm1(-p[6] * b), float.fromhex("0x1.fffffffffffffp-1"))
    fs = min(-math.expm1(-p[7] * s), float.fromhex("0x1.fffffffffffffp-1"))
    thr = p[5] * fb * fs
    return p[0] + (p[1] + p[2] * s) / thr + p[3] * b + p[4] * s


def refit_cases():
    """(meta, b, s, y) with samples concatenated; meta rows carry offsets."""
    rng = np.random.default_rng(77)
    metas, B, S, Y = [], [], [], []

    def add(kind, priors, long_w, short_w, min_s, b, s, y):
        metas.append({"kind": kind, "priors": [float(x) for x in priors], "long_w": int(long_w),
                      "short_w": int(short_w), "min_s": int(min_s), "off": sum(len(x) for x in B),
                      "n": len(b)})
        B.append(np.asarray(b, dtype=np.int64))
        S.append(np.asarray(s, dtype=np.int64))
        Y.append(np.asarray(y, dtype=np.float64))

    def window(truth, n, sigma, decode_frac=0.6, bmax=256):
        b = rng.integers(1, bmax + 1, n)
        s = b.copy()
        pre = rng.random(n) >= decode_frac
        s[pre] = b[pre] + rng.integers(1, 8000, int(pre.sum()))
        y = np.array([_predict(truth, int(bb), int(ss)) for bb, ss in zip(b, s)])
        if sigma > 0:
            y = y * np.exp(sigma * rng.standard_normal(n))
        return b, s, y

    for i in range(12):   # structural refits, full-size windows
        truth = _perturb(rng, [FAST, MEDIUM, SLOW][i % 3])
        n = int(rng.choice([300, 1024, 4096, 5000]))
        b, s, y = window(truth, n, float(rng.choice([0.0, 0.02, 0.05, 0.1])))
        pri = PRIORS if i % 2 == 0 else _perturb(rng, PRIORS)
        add(1, pri, 4096, 64, 256, b, s, y)
    for i in range(6):    # structural, small presets (homogeneous8.json windows 64/16)
        truth = _perturb(rng, FAST)
        b, s, y = window(truth, int(rng.integers(64, 700)), 0.05)
        add(1, PRIORS, int(rng.choice([512, 1024])), 16, 64, b, s, y)
    b, s, y = window(FAST, 1024, 0.05, decode_frac=1.0, bmax=2)   # only tiny decode shapes
    add(1, PRIORS, 4096, 64, 256, b, s, y)
    b = np.full(1024, 200); s = b + 7000                          # saturated in both factors
    add(1, [1.0, 0.0, 1.0, 0.01, 0.001, 10.0, 5.0, 0.5], 4096, 64, 256, b, s,
        [_predict(FAST, 200, 7200)] * 1024)
    add(1, PRIORS, 4096, 64, 2048, *window(FAST, 1000, 0.05))     # below min_structural_samples
    for i in range(30):   # linear refits
        truth = _perturb(rng, [FAST, MEDIUM, SLOW][i % 3])
        sw = int(rng.choice([16, 32, 64]))
        n = int(rng.integers(3, 300))
        pri = PRIORS if i % 3 else _perturb(rng, PRIORS)
        add(0, pri, 4096, sw, 256, *window(truth, n, float(rng.choice([0.0, 0.05]))))
    for i in range(4):    # degenerate design -> rescale fallback
        n = 64
        add(0, PRIORS, 4096, 64, 256, np.full(n, 3), np.full(n, 3), np.full(n, 7.5 + i))
    add(0, PRIORS, 4096, 64, 256, [1, 2], [1, 2], [3.0, 4.0])     # fewer than 5 samples
    add(0, PRIORS, 4096, 64, 256, [4, 4, 4], [4, 5, 6], [1.0, -2.0, 3.0])   # invalid sample
    return metas, np.concatenate(B), np.concatenate(S), np.concatenate(Y)
