"""The library's NCCL path on one GPU (world 1): unique id -> communicator ->
smg_gather_meshes; the gathered rows are the local rows.  The N > 1 host logic
(sharding, ragged padding, rank order) is covered over gloo in
test_shard_gloo.py; this box has one GPU and NCCL refuses two ranks on one device."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_1810_02719_b200")


def test_library_gather_world1(ctx):
    import torch
    from paper_1810_02719_b200 import shard
    comm = shard.LibComm(ctx, 1, 0)
    for total, row in ((5, 7), (64, 3 * 1024)):
        local = torch.arange(total * row, dtype=torch.float64, device="cuda").reshape(total, row)
        out = torch.full((total, row), -1.0, dtype=torch.float64, device="cuda")
        comm.gather(local, out, total, row)
        torch.cuda.synchronize()
        assert torch.equal(out, local)
    comm.close()
