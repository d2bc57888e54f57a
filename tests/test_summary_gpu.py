"""K7 device-side summaries (device/summary.cu) against the reference's
arithmetic (proj/src/metrics.cpp:7-91) restated in Python over the device's
own records: nearest-rank percentiles of the sorted values, the means as left
folds in record order, the SLO-pass fraction — bit-exact. The summary JSON
(which now carries the device's metrics) is compared with the compiled
reference in test_gpu_parity / test_configs_gpu."""
import math

import pytest

from test_gpu_parity import all_cases, device_batch  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu


def _percentile(v, p):  # metrics.cpp:29-38
    v = sorted(v)
    rank = math.ceil(p / 100.0 * len(v))
    return v[max(rank, 1) - 1]


def _host_metrics(recs, ttft_slo, tpot_slo):  # metrics.cpp:40-91
    e2e, ttft, tpot = [], [], []
    ts = ps = 0.0
    n_tp = passed = 0
    for r in recs:
        t = r.first_token_ms - r.arrival_ms
        e = r.completed_ms - r.arrival_ms
        single = r.output_tokens < 2
        tp = 0.0 if single else (r.completed_ms - r.first_token_ms) / float(r.output_tokens - 1)
        e2e.append(e)
        ttft.append(t)
        ts += t
        if not single:
            tpot.append(tp)
            ps += tp
            n_tp += 1
        if t <= ttft_slo and (single or tp <= tpot_slo):
            passed += 1
    n = len(recs)
    return {"completed": n,
            "p50_e2e_ms": _percentile(e2e, 50.0), "p90_e2e_ms": _percentile(e2e, 90.0),
            "p50_ttft_ms": _percentile(ttft, 50.0),
            "p50_tpot_ms": _percentile(tpot, 50.0) if tpot else 0.0,
            "mean_ttft_ms": ts / n, "mean_tpot_ms": ps / n_tp if n_tp else 0.0,
            "slo_attainment_pct": 100.0 * passed / n}


def test_device_metrics_bit_exact(device_batch, all_cases):  # noqa: F811
    names, b = device_batch
    checked = 0
    for i, n in enumerate(names):
        if b.summaries()[i].status != 0:
            continue
        recs = b.records(i)
        if not recs:
            continue
        slo = all_cases[n]["slo"]
        want = _host_metrics(recs, float(slo["ttft_slo_ms"]), float(slo["tpot_slo_ms"]))
        got = b.metrics(i)
        assert got == want, (n, got, want)
        checked += 1
    assert checked >= 20
