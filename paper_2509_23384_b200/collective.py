"""K6 communicator: an NCCL communicator owned by the product library
(nx_nccl_* in include/nx_sched.h), for the one cross-GPU exchange of the
path — the all-gather of per-replica summaries after a sharded sweep. The
unique id travels over any channel the caller has (here torch.distributed's
object broadcast)."""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib

NCCL_ID_BYTES = 128


class NcclComm:
    def __init__(self, unique_id: bytes, nranks: int, rank: int, device: int):
        assert len(unique_id) == NCCL_ID_BYTES
        self._id = C.create_string_buffer(unique_id, NCCL_ID_BYTES)
        h = C.c_void_p()
        check(lib().nx_nccl_comm_init(self._id, nranks, rank, device, C.byref(h)))
        self.handle = h
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(NCCL_ID_BYTES)
        check(lib().nx_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_dist(cls, rank: int, world: int, device: int) -> "NcclComm":
        """Rank 0 makes the id; torch.distributed broadcasts it."""
        import torch.distributed as dist
        box = [cls.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        return cls(box[0], world, rank, device)

    def close(self):
        if self.handle:
            check(lib().nx_nccl_comm_destroy(self.handle))
            self.handle = None
