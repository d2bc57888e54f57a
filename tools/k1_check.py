"""K1 check: device perf_eval vs the CPU oracle (small launch: direct
evaluation; large launch: memo-table path) + timing at 2^26 records."""
import sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np, torch
from paper_2509_23384_b200 import perf_model
from oracle_lib import Port
rows = [perf_model.PROFILES[k] for k in ("fast", "medium", "slow")] + [perf_model.DEFAULT_PRIORS]
port = Port()
for n in (100000, 1 << 22):
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 4, n); b = rng.integers(1, 700, n); s = b + rng.integers(0, 20000, n)
    T, thr = perf_model.eval_host(rows, idx, b, s)
    for k in range(4):
        m = idx == k
        Tr, thr_r = port.perf_eval(list(np.asarray(perf_model._row(rows[k]))), b[m], s[m])
        rel = np.abs(T[m] - Tr) / np.abs(Tr)
        print(n, k, "max rel T", rel.max(), "identical T", np.mean(T[m] == Tr), "identical thr", np.mean(thr[m] == thr_r))
dev = torch.device("cuda")
N = 1 << 26
P = perf_model.profile_table(dev)
g = torch.Generator(device=dev).manual_seed(5)
I = torch.randint(0, P.shape[0], (N,), device=dev, dtype=torch.int32, generator=g)
B = torch.randint(1, 257, (N,), device=dev, dtype=torch.int32, generator=g)
S = B + torch.randint(0, 8192, (N,), device=dev, dtype=torch.int32, generator=g)
out = torch.empty(N, device=dev, dtype=torch.float64)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
stat = torch.zeros(1, dtype=torch.int32, device=dev)
ts = []
for it in range(13):
    flush.fill_(it & 0xff)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); perf_model.eval_device_async(P, I, B, S, out, stat, stream=st); e1.record(st); torch.cuda.synchronize()
    if it >= 3: ts.append(e0.elapsed_time(e1))
t = statistics.mean(ts) / 1e3
print(f"K1: {N/t/1e9:.1f} G rec/s, {N*20/t/1e9:.0f} GB/s, {t*1e6:.0f} us, status {int(stat.item())}")
