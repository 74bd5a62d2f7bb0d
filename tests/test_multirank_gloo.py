"""Multi-rank host logic on CPU (gloo, world_size 2 and 4): node ownership (reading R17) and
the cross-rank node sum used by the binding, applied to per-rank partial projectors
computed by the oracle: the all-reduced partials equal the single-rank projector."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import oracle
    import synth
    from paper_1404_2891_b200.feast import allreduce_node_sum
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = synth.make_pencil("C2", n=72, m0=6)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    j0, j1 = synth.node_owner_range(len(z), rank, world)
    part = torch.from_numpy(oracle.project(P.A, P.B, P.X0, z, w, j0, j1).copy())
    allreduce_node_sum(part)
    # max-over-ranks timing reduction used by bench.py
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(out, part.numpy())
        assert t.item() == float(world)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_node_sum_across_ranks(tmp_path, world):
    import oracle
    import synth
    out = str(tmp_path / "q.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    P = synth.make_pencil("C2", n=72, m0=6)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    full = oracle.project(P.A, P.B, P.X0, z, w)
    got = np.load(out)
    assert np.linalg.norm(got - full) / np.linalg.norm(full) < 1e-13
