#!/usr/bin/env python3
"""NexusSched hot-path benchmark: scheduling decisions/s (routes + batches).

Workload (BASELINE.json config 5): the arrival-rate x seed x router-policy
sweep of 8-engine heterogeneous LENS+PRISM replicas (2000 sharegpt requests
each). Replicas are independent, so every GPU owns a fixed shard of
`--replicas-per-gpu` (default 512) replicas of the interleaved 4096-replica
grid — rank k runs grid rows [k*R, (k+1)*R) — and N GPUs run N*R replicas
("scaling": "weak"; N=8 is exactly the 4096-replica sweep). One step = one
launch of the device lockstep kernel over the rank's whole shard, inputs
resident in HBM. The single collective is the end-of-run NCCL all-gather of
per-replica summaries (K6).

  value : decisions / device time of the K timed launches (max over ranks)
  e2e   : same metric through the C-ABI with host buffers each step
          (pinned H2D of the traces + descriptors, launch, D2H of results)
  --impl reference : the reference C++ simulator (oracle/_ref, compiled
          unmodified from /root/reference/proj/src) on the host cores, same
          workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "scheduling decisions/sec (routes+batches) at 1/2/4/8 B200; % HBM roofline"
UNIT = "decisions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["nx", "reference"], default="nx")
    ap.add_argument("--replicas-per-gpu", type=int, default=512)
    ap.add_argument("--requests", type=int, default=2000)
    ap.add_argument("--cpu-sample", type=int, default=512,
                    help="replicas of the rank-0 shard timed for cpu_baseline (and parity-checked)")
    ap.add_argument("--no-configs", action="store_true", help="skip BASELINE configs 1-4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-operators", action="store_true", help="skip the batched K2/K3/K4 lines")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the in-run ncu DRAM-traffic probe (roofline.traffic from profiles/ instead)")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def shard_configs(rank: int, per_gpu: int, n_req: int):
    from paper_2509_23384_b200 import workloads as W
    total = per_gpu * (rank + 1)
    grid = W.sweep_configs(n_replicas=min(4096, max(total, 1)), n=n_req)
    if total > len(grid):  # beyond the 4096 grid: extend with further seeds
        extra = []
        seed = 65
        while len(grid) + len(extra) < total:
            for rate in W.SWEEP_RATES:
                for pol in W.SWEEP_POLICIES:
                    extra.append(W.sweep_replica(rate, seed, pol, n_req))
            seed += 1
        grid = grid + extra
    return grid[rank * per_gpu:(rank + 1) * per_gpu]


def workload_desc(per_gpu: int, n_req: int, n_gpus: int) -> dict:
    return {
        "workload": (f"config5 sweep shard: {per_gpu} replicas/GPU of the rate x seed x policy grid "
                     f"(16 rates 10..47.5 req/s x 4 router policies prism/round_robin/least_loaded/"
                     f"latency_based x seeds), 8 heterogeneous engines (2 fast/3 medium/3 slow), "
                     f"LENS scheduler + online learner, {n_req} sharegpt requests per replica"),
        "replicas_per_gpu": per_gpu,
        "replicas_total": per_gpu * n_gpus,
        "requests_per_replica": n_req,
        "l2": "flushed between timed steps (256 MiB device write)",
        "parallelism": f"replica-sharded dp{n_gpus}",
    }


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------- roofline
def algorithmic_bytes(batch, n_rep: int, n_eng: int = 8) -> int:
    """SURVEY.md §8(d) compulsory bytes, from the device work counters."""
    total = 0
    sums = batch.summaries()
    for r in range(n_rep):
        w = batch.work(r)
        steps, sum_b, win, lin, struct = w[0], w[1], w[2], w[3], w[4]
        total += sums[r].arrived * (48 * n_eng + 36)       # K3 per route
        total += steps * (96 + 24) + 4 * win + 8 * sum_b     # K2 per batch decision
        total += 32 * sum_b + steps * (64 + 32)              # K5 per executed step
        total += 16 * lin + 16 * struct                      # K4 refits (window reads)
    return total


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def k1_model_eval(torch, dev) -> dict:
    """K1 perf-model evaluator on 2^26 streamed records (HBM-bound)."""
    from paper_2509_23384_b200 import perf_model
    n = 1 << 26
    g = torch.Generator(device=dev).manual_seed(5)
    params = perf_model.profile_table(dev)          # fast/medium/slow + priors
    idx = torch.randint(0, params.shape[0], (n,), device=dev, dtype=torch.int32, generator=g)
    b = torch.randint(1, 257, (n,), device=dev, dtype=torch.int32, generator=g)
    s = b + torch.randint(0, 8192, (n,), device=dev, dtype=torch.int32, generator=g)
    out = torch.empty(n, device=dev, dtype=torch.float64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    times = []
    for it in range(8):
        flush.fill_(it & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        perf_model.eval_device_async(params, idx, b, s, out, status, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if it >= 3:
            times.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.mean(times)
    if int(status.item()) != 0:
        raise RuntimeError("K1 flagged invalid records")
    byts = n * (4 + 4 + 4 + 8)
    pk, src = peaks()
    return {"kernel": "perf_eval_kernel (K1, fp64 deterministic)", "records": n,
            "records_per_s": n / t, "ms": t * 1e3,
            "roofline": {"bound": "hbm", "achieved": byts / t / 1e9, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": byts / t / 1e9 / pk["hbm_gbs"],
                         "traffic": traffic("perf_eval_kernel"), "peak_source": src,
                         "bytes_per_record": 20}}


TRAFFIC_FILE = "r02_traffic.json"
TRAFFIC_SOURCE = (f"profiles/{TRAFFIC_FILE}: dram__bytes_read.sum + dram__bytes_write.sum of one "
                  "ncu --set full capture of this build (not re-measured in this run)")


_TRAFFIC = {}  # measured in this run (probe_traffic), else the committed capture


def traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`:
    measured in this run by the ncu probe when it ran, else from the committed
    ncu --set full capture of the current build."""
    if kernel in _TRAFFIC:
        return _TRAFFIC[kernel]
    try:
        t = json.loads((ROOT / "profiles" / TRAFFIC_FILE).read_text())
        return t[kernel]["traffic_bytes_per_launch"]
    except Exception:
        return None


def probe_traffic(args) -> str:
    """One launch of the bench-shard simulation and of K1 under
    `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` (a child
    process: a profiled launch is never a timed one), same box, same build.
    Fills _TRAFFIC; returns a description for roofline.traffic_source."""
    import shutil
    import subprocess
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).exists():
        return TRAFFIC_SOURCE + " (ncu not found for the in-run probe)"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
           "--print-units", "base", "--csv", "-k", "regex:nx_sim_kernel|perf_eval_kernel",
           sys.executable, str(ROOT / "bench.py"), "--traffic-probe",
           "--replicas-per-gpu", str(args.replicas_per_gpu), "--requests", str(args.requests)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600).stdout
    except Exception as exc:  # noqa: BLE001 — the committed capture stays the fallback
        return TRAFFIC_SOURCE + f" (in-run probe failed: {exc!r})"
    import csv
    import io
    got = {}
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 5]
    if rows:
        hdr = rows[0]
        try:
            kn, mn, mv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
            for r in rows[1:]:
                k = "nx_sim_kernel" if "nx_sim_kernel" in r[kn] else (
                    "perf_eval_kernel" if "perf_eval_kernel" in r[kn] else None)
                if k and r[mn].startswith("dram__bytes_"):
                    got.setdefault(k, {})[r[mn]] = float(r[mv].replace(",", ""))
        except ValueError:
            got = {}
    for k, m in got.items():
        if len(m) == 2:
            _TRAFFIC[k] = int(sum(m.values()))
    if not _TRAFFIC:
        return TRAFFIC_SOURCE + " (in-run probe returned no counters)"
    return ("measured in this run: dram__bytes_read.sum + dram__bytes_write.sum of one launch of the "
            "same workload under ncu --clock-control none (child process, not timed)")


def traffic_probe_child(args):
    """The ncu child of probe_traffic: one shard launch, one K1 launch."""
    import torch
    from paper_2509_23384_b200 import perf_model, sim
    dev = torch.device("cuda", 0)
    b = sim.Batch(shard_configs(0, args.replicas_per_gpu, args.requests))
    b.run()
    b.close()
    n = 1 << 26
    g = torch.Generator(device=dev).manual_seed(5)
    params = perf_model.profile_table(dev)
    idx = torch.randint(0, params.shape[0], (n,), device=dev, dtype=torch.int32, generator=g)
    bb = torch.randint(1, 257, (n,), device=dev, dtype=torch.int32, generator=g)
    ss = bb + torch.randint(0, 8192, (n,), device=dev, dtype=torch.int32, generator=g)
    out = torch.empty(n, device=dev, dtype=torch.float64)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    perf_model.eval_device_async(params, idx, bb, ss, out, status, stream=torch.cuda.current_stream(dev))
    torch.cuda.synchronize(dev)


def baseline_configs_line(torch, local: int) -> dict:
    """BASELINE configs 1-4 at their stated sizes: one
    device batch of the five single-replica runs, each replica's own device
    time (%globaltimer begin/end) -> decisions/s, next to the reference
    simulator (oracle/_ref) on one host thread per config, and the parity of
    the two (event hash + decisions). Single replicas do not shard
    ("replicas only"): a replica's event loop is sequential."""
    import tempfile
    from paper_2509_23384_b200 import sim, workloads as W
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Port, Ref, ref_available
    from concurrent.futures import ThreadPoolExecutor
    td = tempfile.mkdtemp(prefix="nx_cfg_")
    cfgs = W.baseline_configs(td, sim.synth_generate)
    names = list(cfgs)
    chk = Ref() if ref_available() else Port()

    def ref_one(c):
        t0 = time.perf_counter()
        r = chk.run(c)
        return r, time.perf_counter() - t0

    with ThreadPoolExecutor(max_workers=len(names)) as ex:
        futs = {n: ex.submit(ref_one, cfgs[n]) for n in names}
        b = sim.Batch([cfgs[n] for n in names], device=local)
        b.upload()
        b.launch()
        b.download()
        b.synchronize()
        launch_ms = b.kernel_ms()
        sums = b.summaries()
        out = {}
        for i, n in enumerate(names):
            t0, t1 = b.timeline(i)
            dev_s = max(1e-9, (t1 - t0) / 1e9)
            want, ref_s = futs[n].result()
            out[n] = {"decisions": sums[i].decisions, "device_s": dev_s,
                      "device_decisions_per_s": sums[i].decisions / dev_s,
                      "reference_s": ref_s, "reference_decisions_per_s": want["decisions"] / ref_s,
                      "event_hash_equal": f"{sums[i].event_hash:016x}" == want["event_hash"],
                      "decisions_equal": sums[i].decisions == want["decisions"]}
    b.close()
    return {"launch_ms": launch_ms, "reference_kind": "reference" if ref_available() else "port",
            "reference_threads": "one host thread per config, all five concurrently",
            "note": "single replicas: sequential event loops, run side by side in one launch",
            "per_config": out}


def operators(torch, dev) -> dict:
    """The batched per-decision operators on device-resident batches:
    K2 nx_lens_schedule (LENS decisions/s), K3 nx_prism_route (routes/s,
    PRISM with echo), K4 nx_refit (structural refits/s on 4096-sample
    windows). Device time per launch with CUDA events, after warm-up."""
    import ctypes as C
    import numpy as np
    from paper_2509_23384_b200 import abi, lens, learner
    from paper_2509_23384_b200._lib import check, lib
    rng = np.random.default_rng(11)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, reps=5):
        ts = []
        for it in range(reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if it >= 2:
                ts.append(e0.elapsed_time(e1) / 1e3)
        return statistics.mean(ts)

    def dev_bytes(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(dev)

    out = {}
    # K2: LENS decisions over queues shaped like the sweep's engines
    n = 1 << 17
    P = np.zeros(n, dtype=abi.LENS_PROBLEM)
    R = rng.integers(0, 64, n)
    W = rng.integers(0, 64, n)
    off = np.concatenate([[0], np.cumsum(W)[:-1]])
    fast = [4.0, 0.0, 1.0, 0.08, 0.0004, 20.0, 4.0, 0.05]
    for k, v in zip(("ttft_slo_ms", "tpot_slo_ms", "alpha_ms", "beta", "l_bar", "td_min_ms",
                     "eps_ratio", "q_ref", "m_max", "q_max", "n_search_iters"),
                    (2000.0, 50.0, 4000.0, 40.0, 128.0, 2.0, 0.05, 16.0, 8192, 256, 10)):
        P[k] = v
    P["params"] = fast
    P["n_run"], P["n_wait"], P["wait_off"] = R, W, off
    rem = np.exp(rng.uniform(0, np.log(2000), int(W.sum()))).astype(np.int32) + 1
    dP, dR = dev_bytes(P), torch.from_numpy(rem).to(dev)
    dPl = torch.empty(n * abi.LENS_PLAN.itemsize, dtype=torch.uint8, device=dev)
    dA = torch.empty(rem.size, dtype=torch.int32, device=dev)
    t = timed(lambda: check(lib().nx_lens_schedule_dev(dP.data_ptr(), n, dR.data_ptr(), rem.size,
                                                       dPl.data_ptr(), dA.data_ptr(),
                                                       C.c_void_p(stream.cuda_stream))))
    plans = np.frombuffer(dPl.cpu().numpy().tobytes(), dtype=abi.LENS_PLAN)
    if (plans["status"] != 0).any():
        raise RuntimeError("nx_lens_schedule: problem errors")
    out["lens_decisions_per_s"] = n / t
    # the same batch in NX_FAST_FP32 (float probes; decisions may differ)
    t32 = timed(lambda: check(lib().nx_lens_schedule_mode_dev(dP.data_ptr(), n, dR.data_ptr(), rem.size,
                                                              dPl.data_ptr(), dA.data_ptr(), 1,
                                                              C.c_void_p(stream.cuda_stream))))
    p32 = np.frombuffer(dPl.cpu().numpy().tobytes(), dtype=abi.LENS_PLAN)
    out["lens_fp32_decisions_per_s"] = n / t32
    out["lens_fp32_same_plan_frac"] = float(np.mean((p32["b"] == plans["b"]) & (p32["s"] == plans["s"])))
    out["lens_batch"] = f"{n} decisions, |run| U[0,64), |wait| U[0,64)"
    # K3: routers of 8 engines, 32 PRISM routes each (sequential within a group)
    g, e, m = 1 << 14, 8, 32
    G = np.zeros(g, dtype=abi.ROUTE_GROUP)
    G["weights"] = [1.0, 1.0, 1.0, 1.0]
    G["beta_aff"], G["latency_knee"], G["load_half_ms"] = 1.5, 0.5, 50.0
    G["capacity_headroom"], G["staleness_limit_ms"], G["ttft_slo_ms"] = 2.0, 1000.0, 2000.0
    G["l_bar_ema"], G["policy"], G["n_engines"], G["n_requests"], G["n_sessions"] = 128.0, 0, e, m, 64
    G["engine_off"] = np.arange(g) * e
    G["request_off"] = np.arange(g) * m
    G["session_off"] = np.arange(g) * 64
    Rp = np.zeros(g * e, dtype=abi.ENGINE_REPORT)
    Rp["l_hat_ms"] = rng.uniform(0, 3000, g * e)
    Rp["w_load_tokens"] = rng.uniform(0, 50000, g * e)
    Rp["m_free_tokens"] = rng.uniform(0, 2e5, g * e)
    Rp["p_max"] = rng.uniform(5, 20, g * e)
    Rp["reported_at_ms"] = 0.0
    Rp["has_report"], Rp["static_weight"] = 1, 1.0
    Rp["engine_id"] = np.tile(np.arange(e), g)
    Q = np.zeros(g * m, dtype=abi.ROUTE_REQUEST)
    Q["now_ms"] = rng.uniform(0, 900, g * m)
    Q["prompt_len"] = rng.integers(1, 4000, g * m)
    Q["session"] = rng.integers(0, 64, g * m)
    dG, dRp, dQ = dev_bytes(G), dev_bytes(Rp), dev_bytes(Q)
    dS = torch.full((g * 64,), -1, dtype=torch.int32, device=dev)
    dD = torch.empty(g * m * abi.ROUTE_DECISION.itemsize, dtype=torch.uint8, device=dev)
    dSt = torch.empty(g, dtype=torch.int32, device=dev)
    t = timed(lambda: check(lib().nx_prism_route_dev(dG.data_ptr(), g, dRp.data_ptr(), dQ.data_ptr(),
                                                     dS.data_ptr(), dD.data_ptr(), dSt.data_ptr(),
                                                     C.c_void_p(stream.cuda_stream))))
    if int((dSt != 0).sum().item()):
        raise RuntimeError("nx_prism_route: group errors")
    out["prism_routes_per_s"] = g * m / t
    t32 = timed(lambda: check(lib().nx_prism_route_mode_dev(dG.data_ptr(), g, dRp.data_ptr(), dQ.data_ptr(),
                                                            dS.data_ptr(), dD.data_ptr(), dSt.data_ptr(), 1,
                                                            C.c_void_p(stream.cuda_stream))))
    out["prism_fp32_routes_per_s"] = g * m / t32
    out["prism_batch"] = f"{g} routers x {m} sequential routes, {e} engines each"
    # K4: structural refits on 4096-sample windows
    nr, wl = 1024, 4096
    b = rng.integers(1, 257, nr * wl).astype(np.int32)
    s_ = (b + np.where(rng.random(nr * wl) < 0.4, rng.integers(1, 8000, nr * wl), 0)).astype(np.int32)
    bd, sd = b.astype(np.float64), s_.astype(np.float64)
    fb = np.minimum(-np.expm1(-4.0 * bd), 1.0)
    fs = np.minimum(-np.expm1(-0.05 * sd), 1.0)
    y = (4.0 + sd / (20.0 * fb * fs) + 0.08 * bd + 4e-4 * sd) * np.exp(0.05 * rng.standard_normal(nr * wl))
    RP = np.zeros(nr, dtype=abi.REFIT_PROBLEM)
    RP["params"] = [5.0, 0.0, 1.0, 0.1, 0.001, 20.0, 0.1, 0.02]
    RP["long_window"], RP["short_window"], RP["min_structural_samples"] = wl, 64, 256
    RP["sample_off"], RP["n_samples"] = np.arange(nr) * wl, wl
    dRP, dB, dS2, dY = dev_bytes(RP), torch.from_numpy(b).to(dev), torch.from_numpy(s_).to(dev), \
        torch.from_numpy(y).to(dev)
    dO = torch.empty(nr * abi.REFIT_RESULT.itemsize, dtype=torch.uint8, device=dev)
    t = timed(lambda: check(lib().nx_refit_dev(learner.STRUCTURAL, dRP.data_ptr(), nr, dB.data_ptr(),
                                               dS2.data_ptr(), dY.data_ptr(), wl, dO.data_ptr(),
                                               C.c_void_p(stream.cuda_stream))), reps=3)
    res = np.frombuffer(dO.cpu().numpy().tobytes(), dtype=abi.REFIT_RESULT)
    if (res["status"] != 0).any():
        raise RuntimeError("nx_refit: problem errors")
    out["structural_refits_per_s"] = nr / t
    out["refit_batch"] = f"{nr} OnlineLearner::update_structural on {wl}-sample windows"
    return out


# ---------------------------------------------------------------------------- arms
def balanced_prefix(n: int, k: int):
    """Indices of a sample of k replicas with every rate x policy cell equally
    represented: the shard grid is seed-major with all 16 rates x 4 router
    policies inside each seed (workloads.sweep_configs), so whole 64-replica
    seed blocks from the front of the shard are exactly balanced (a strided
    pick with step 4 would alias onto a single policy)."""
    k = max(1, min(n, 64 * math.ceil(max(1, k) / 64)))
    return list(range(k))


def longest_first(cfgs, idx):
    """Replica indices ordered longest expected first (lowest arrival rate:
    most steps), so a host thread pool ends on short replicas."""
    return sorted(idx, key=lambda i: cfgs[i]["workload"]["rate"])


def cpu_reference_rate(cfgs, threads: int, detail: bool = False):
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Port, Ref, ref_available
    checker = Ref() if ref_available() else Port()
    kind = "reference" if ref_available() else "port"
    dec, hashes, wall = checker.run_batch(cfgs, threads)
    if detail:
        return sum(dec) / wall, kind, wall, sum(dec), dec, hashes
    return sum(dec) / wall, kind, wall, sum(dec)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cfgs = shard_configs(0, args.replicas_per_gpu, args.requests)
    # ~8 replicas per host thread in whole rate x policy blocks, longest
    # expected first: the dynamic queue then ends with short replicas instead
    # of idling cores behind a long one
    sample = [cfgs[i] for i in longest_first(cfgs, balanced_prefix(len(cfgs), 8 * threads))]
    rates = []
    for i in range(args.warmup + args.steps):
        r, kind, wall, dec = cpu_reference_rate(sample, threads)
        if i >= args.warmup:
            rates.append((r, wall, dec))
    tot_dec = sum(x[2] for x in rates)
    tot_wall = sum(x[1] for x in rates)
    value = tot_dec / tot_wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_wall / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_desc(args.replicas_per_gpu, args.requests, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{len(sample)} replicas of the rank-0 shard per step (whole "
                                   f"seed blocks: every rate x policy cell equally), longest first, "
                                   f"one std::thread per host core"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_nx(args):
    import torch
    import torch.distributed as dist

    from paper_2509_23384_b200 import sim

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # NX_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0 with gloo for
    # the host-side plumbing, so the N>1 path runs on a one-GPU box (NCCL
    # refuses two ranks on one device)
    one_dev = os.environ.get("NX_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = "gloo" if one_dev else "nccl"
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if backend == "gloo" else dev

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    cfgs = shard_configs(rank, args.replicas_per_gpu, args.requests)
    batch = sim.Batch(cfgs, device=local, host_threads=os.cpu_count())
    batch.upload()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    for i in range(args.warmup):
        batch.launch()
        batch.synchronize()
    batch.download()
    batch.synchronize()
    sums = batch.summaries()
    bad = [i for i, s in enumerate(sums) if s.status != 0]
    if bad:
        raise RuntimeError(f"rank {rank}: {len(bad)} replicas failed (first site {sums[bad[0]].err_site})")
    decisions_step = sum(s.decisions for s in sums)

    barrier()
    kernel_s = 0.0
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            torch.cuda.synchronize(dev)
            batch.launch()
            batch.synchronize()
            kernel_s += batch.kernel_ms() / 1e3
    barrier()
    t_dev = max_over_ranks(kernel_s)
    total_dec = sum_over_ranks(decisions_step * args.steps)
    value = total_dec / t_dev

    # e2e through the C-ABI with host buffers: workload generation on the
    # host (as inside the reference's run_simulation clock), pinned H2D,
    # launch, D2H of the results, per-replica summaries
    # (pipelined as a caller running batch after batch would: the next
    # step's workload is built on the host while the device runs this one;
    # every step still pays its own synthesis, H2D, launch and D2H)
    e2e = None
    if not args.no_e2e:
        barrier()
        t0 = time.perf_counter()
        batch.rebuild_workloads(os.cpu_count())
        for i in range(args.steps):
            batch.upload()
            batch.launch()
            batch.download()
            if i + 1 < args.steps:
                batch.rebuild_workloads(os.cpu_count())  # waits for this step's H2D only
            batch.synchronize()
            e2e_sums = batch.summaries()
        wall = time.perf_counter() - t0
        if sum(x.decisions for x in e2e_sums) != decisions_step:
            raise RuntimeError("e2e run diverged from the timed launches")
        barrier()
        h2d, d2h = batch.io_bytes()
        e2e_t = max_over_ranks(wall)
        e2e = {"value": total_dec / e2e_t, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    # K6: one NCCL all-gather of the per-replica summaries (the only exchange),
    # over the product library's own communicator (nx_nccl_*); torch's
    # all-gather only if that communicator cannot be built
    gathered = None
    if world > 1:
        nbytes = batch.summaries_nbytes()
        out = torch.empty(nbytes * world, dtype=torch.uint8, device=dev)
        buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        batch.copy_summaries(buf.data_ptr())
        if backend == "nccl":
            try:
                from paper_2509_23384_b200.collective import NcclComm
                comm = NcclComm.from_torch_dist(rank, world, local)
                batch.gather_summaries(comm, out.data_ptr())
                batch.synchronize()
                comm.close()
                gather_via = "nx_sim_gather_summaries (ncclAllGather)"
            except Exception as exc:  # noqa: BLE001
                dist.all_gather_into_tensor(out, buf)
                torch.cuda.synchronize(dev)
                gather_via = f"torch all_gather ({exc!r})"
        else:  # gloo: host copies of the same bytes
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, buf.cpu())
            out.copy_(torch.cat(parts))
            gather_via = "torch.distributed gloo all_gather of host copies (one-device test mode)"
        # every rank's records arrived intact: this rank's slice is its own
        if not torch.equal(out[rank * nbytes:(rank + 1) * nbytes], buf):
            raise RuntimeError("summary gather corrupted this rank's records")
        gathered = world * len(cfgs)

    # roofline of the dominant kernel (nx_sim_kernel), from device work counters
    traffic_source = TRAFFIC_SOURCE
    if rank == 0 and world == 1 and not args.no_traffic:
        traffic_source = probe_traffic(args)
    pk, src = peaks()
    alg = algorithmic_bytes(batch, len(cfgs))
    per_launch_s = kernel_s / args.steps
    achieved = alg / per_launch_s / 1e9

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_dev / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(args.replicas_per_gpu, args.requests, world),
            "decisions_per_step": total_dec / args.steps,
            "gpu_launches": 2 * args.steps,  # nx_sim_kernel + nx_summarize_kernel per launch
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic("nx_sim_kernel"),
                         "traffic_source": traffic_source,
                         "kernel": "nx_sim_kernel", "peak_source": src,
                         "algorithmic_bytes_per_launch": alg,
                         "limiter": "latency, not HBM: a replica's critical path is the sum over its "
                                    "arrival windows of the slowest engine warp's events (structural "
                                    "refits about half of it); the achieved GB/s is algorithmic bytes "
                                    "over that time (DESIGN.md §5)"},
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if gathered is not None:
            line["gathered_summaries"] = gathered
            line["gather_via"] = gather_via
        try:
            line["model_eval"] = k1_model_eval(torch, dev)
        except Exception as exc:  # keep the headline line even if K1 fails
            line["model_eval"] = {"error": repr(exc)}
        if not args.no_operators:
            try:
                line["operators"] = operators(torch, dev)
            except Exception as exc:
                line["operators"] = {"error": repr(exc)}
        if not args.no_cpu_baseline:
            # the whole rank-0 shard through the reference on every host core,
            # longest expected first (lowest rate), as in the reference arm
            idx = longest_first(cfgs, balanced_prefix(len(cfgs), args.cpu_sample))
            sample = [cfgs[i] for i in idx]
            rate, kind, wall, dec, rdec, rhash = cpu_reference_rate(sample, os.cpu_count() or 1, detail=True)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": kind,
                                    "sample": f"{len(sample)} replicas of the rank-0 shard (every rate x "
                                              f"policy cell), longest first, {dec} decisions in {wall:.1f} s"}
            # the same replicas, checked against the timed device run: the event
            # hash fingerprints every routing choice, batch composition and time
            dsum = batch.summaries()
            pol = [cfgs[i]["router"]["policy"] for i in idx]
            line["cpu_baseline"]["parity"] = {
                "replicas": len(idx),
                "event_hash_equal": sum(int(dsum[i].event_hash == h) for i, h in zip(idx, rhash)),
                "decisions_equal": sum(int(dsum[i].decisions == d) for i, d in zip(idx, rdec)),
                "per_policy": {p: sum(int(x == p) for x in pol) for p in sorted(set(pol))}}
        if not args.no_configs:
            try:
                line["configs"] = baseline_configs_line(torch, local)
            except Exception as exc:  # noqa: BLE001 — keep the headline line
                line["configs"] = {"error": repr(exc)}
        print(json.dumps(line), flush=True)
    batch.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.traffic_probe:
        traffic_probe_child(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_nx(args)


if __name__ == "__main__":
    main()
