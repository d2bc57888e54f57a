"""The N>1 product path on one GPU: world_size 2, both ranks on cuda:0.

* Each rank runs its `bench.shard_configs` shard through _nxsched.so, the raw
  NxReplicaOut records (the K6 payload, nx_sim_copy_summaries) are exchanged
  with gloo over host copies, and the gathered table must equal, byte for
  byte, a single-process run over the union of the shards (only the
  %globaltimer stamps of each record may differ).
* `bench.py --gpus 2` under torchrun (NX_BENCH_ONE_DEVICE=1: gloo plumbing,
  since NCCL refuses two ranks on one device) prints one complete line:
  value, e2e, roofline, clocks, cpu_baseline with its core count and the
  summary gather.
Reference: proj/src/sim.cpp:608-642 (the sweep the shards partition);
SURVEY.md §8(e).
"""
import importlib.util
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REC_BYTES = 280
STAMP = slice(240, 256)  # NxReplicaOut.t_begin_ns, t_end_ns (nx_layout.h)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench():
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _records(batch):
    import torch
    n = batch.summaries_nbytes()
    assert n == batch.n * REC_BYTES
    buf = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    batch.copy_summaries(buf.data_ptr())
    return buf.cpu()


def _worker(rank, world, port, per_rank, n_req, out_path):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    from paper_2509_23384_b200 import sim
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfgs = _bench().shard_configs(rank, per_rank, n_req)
    b = sim.Batch(cfgs, device=0).run()
    mine = _records(b)
    b.close()
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)  # the single result exchange
    if rank == 0:
        torch.save(torch.cat(parts), out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_through_the_library_equal_one_process(tmp_path):
    import torch
    import torch.multiprocessing as mp
    from paper_2509_23384_b200 import sim
    world, per_rank, n_req = 2, 8, 200
    out_path = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(world, _free_port(), per_rank, n_req, out_path), nprocs=world, join=True)
    got = torch.load(out_path).numpy().reshape(-1, REC_BYTES).copy()
    union = _bench().shard_configs(0, world * per_rank, n_req)
    b = sim.Batch(union, device=0).run()
    want = _records(b).numpy().reshape(-1, REC_BYTES).copy()
    sums = b.summaries()
    b.close()
    assert got.shape == want.shape == (world * per_rank, REC_BYTES)
    assert all(s.status == 0 for s in sums)
    got[:, STAMP] = 0
    want[:, STAMP] = 0
    diff = sorted(set(np.nonzero(got != want)[1].tolist()))
    assert np.array_equal(got, want), f"differing byte offsets {diff}"

    # the records carry the event hashes the single-process run reports
    eh = got[:, 40:48].copy().view(np.uint64).ravel()
    assert [int(x) for x in eh] == [s.event_hash for s in sums]


def test_bench_two_ranks_prints_a_complete_line():
    env = dict(os.environ, NX_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--replicas-per-gpu", "8",
           "--requests", "150", "--no-operators", "--no-configs", "--cpu-sample", "8"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["replicas_total"] == 16
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    for k in ("roofline", "clocks", "cpu_baseline", "gather_via", "gathered_summaries", "gpu_launches"):
        assert k in line, k
    assert line["gathered_summaries"] == 16
    cb = line["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["parity"]["event_hash_equal"] == cb["parity"]["replicas"]
