"""Per-call latency of the scalar drop-in calls (each one a device round
trip) vs their batched forms."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_23384_b200 import perf_model as pm, lens
p = pm.PROFILES["fast"]
for _ in range(50):
    pm.predict_latency(p, (4, 100))
n = 2000
t0 = time.perf_counter()
for i in range(n):
    pm.predict_latency(p, (4, 100 + i))
t1 = time.perf_counter()
print(f"predict_latency (scalar, ctypes): {1e6 * (t1 - t0) / n:.1f} us/call")
rows = [p]
N = 1 << 20
rng = np.random.default_rng(1)
b = rng.integers(1, 256, N); s = b + rng.integers(0, 8000, N); idx = np.zeros(N, dtype=np.int64)
pm.eval_host(rows, idx, b, s)
t0 = time.perf_counter()
for _ in range(5):
    pm.eval_host(rows, idx, b, s)
t1 = time.perf_counter()
print(f"predict_latency batched from host arrays (2^20 records incl. H2D/D2H): {1e9 * (t1 - t0) / 5 / N:.2f} ns/record")
# one LENS decision per call (schedule_step) over a small queue
R = [lens.Request(id=i, prompt_len=64, prefilled=64) for i in range(8)]
Wq = [lens.Request(id=100 + i, prompt_len=300 + 17 * i) for i in range(16)]
args = (Wq, R, lens.SLOSpec(), lens.TradeoffModel(), p, lens.SchedulerConfig())
for _ in range(20):
    lens.schedule_step(*args)
m = 500
t0 = time.perf_counter()
for _ in range(m):
    lens.schedule_step(*args)
t1 = time.perf_counter()
print(f"schedule_step (scalar, ctypes, 8 running + 16 waiting): {1e6 * (t1 - t0) / m:.1f} us/call")
# one PRISM routing decision per call (Router::route) over 8 engines
from paper_2509_23384_b200 import router
rt = router.Router(router.RouterConfig(), 2000.0)
for e in range(8):
    rt.register_engine(e)
    rt.on_report(e, 100.0 * e, 1000.0 * e, 50000.0, 20.0, 0.0, e)
for _ in range(20):
    rt.route(500, "s1", 1.0)
m = 500
t0 = time.perf_counter()
for i in range(m):
    rt.route(500 + i, f"s{i % 16}", 1.0 + i)
t1 = time.perf_counter()
print(f"Router::route (scalar, ctypes, 8 engines): {1e6 * (t1 - t0) / m:.1f} us/call")
