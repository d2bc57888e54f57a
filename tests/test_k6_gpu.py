"""K6: the product library's NCCL communicator and summary all-gather
(nx_nccl_*, nx_sim_gather_summaries) on one GPU (nranks = 1: the gathered
buffer is this rank's summaries). Multi-rank shard + gather logic is covered
with gloo in test_multiproc.py."""
import pytest

from cases import static_cases

pytestmark = pytest.mark.gpu


def test_single_rank_gather_returns_this_ranks_summaries():
    import torch
    from paper_2509_23384_b200 import sim
    from paper_2509_23384_b200.collective import NcclComm
    c = static_cases()
    b = sim.Batch([c["c1_small"], c["het_prism"]]).run()
    try:
        n = b.summaries_nbytes()
        mine = torch.empty(n, dtype=torch.uint8, device="cuda")
        b.copy_summaries(mine.data_ptr())
        comm = NcclComm(NcclComm.unique_id(), 1, 0, 0)
        out = torch.zeros(n, dtype=torch.uint8, device="cuda")
        b.gather_summaries(comm, out.data_ptr())
        b.synchronize()
        comm.close()
        assert torch.equal(out, mine)
    finally:
        b.close()
