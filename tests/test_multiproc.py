"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path: each rank
owns a shard of the replica sweep (bench.shard_configs), computes its shard's
per-replica results, and one all-gather of fixed-size summary records is the
only exchange. Rank 0 checks the gathered table equals a
single-process run over the whole sweep. The per-rank compute here is the CPU
oracle (no GPU in this container); on the box the same sharding drives the
device kernel and the gather runs over NCCL."""
import importlib.util
import os
import socket
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


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


def _worker(rank, world, port, per_rank, n_req, out_path):
    import sys
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Port
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfgs = _bench().shard_configs(rank, per_rank, n_req)
    dec, eh, _ = Port().run_batch(cfgs, 2)
    rec = torch.tensor([[d, int(h) & 0x7FFFFFFFFFFFFFFF, int(h) >> 63] for d, h in zip(dec, eh)],
                       dtype=torch.int64)
    out = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(out, rec)  # the single result gather
    if rank == 0:
        torch.save(torch.cat(out), out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sweep_gather_matches_single_process(tmp_path):
    import sys
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Port
    world, per_rank, n_req = 2, 4, 120
    out_path = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(world, _free_port(), per_rank, n_req, out_path), nprocs=world, join=True)
    gathered = torch.load(out_path)
    full = _bench().shard_configs(0, world * per_rank, n_req)
    dec, eh, _ = Port().run_batch(full, 2)
    want = torch.tensor([[d, int(h) & 0x7FFFFFFFFFFFFFFF, int(h) >> 63] for d, h in zip(dec, eh)],
                        dtype=torch.int64)
    assert torch.equal(gathered, want)
