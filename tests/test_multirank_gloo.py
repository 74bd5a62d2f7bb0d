"""Multi-rank host logic on CPU (gloo, world_size 2 and 4): node ownership (reading R17) and the
cross-rank node sum as the library performs it — through the all-reduce callback the
binding registers (paper_1404_2891_b200.feast.make_allreduce_callback), handed a raw pointer to one
flat float64 block, as feast_project hands it the packed [Q | QL] staging block.  The per-rank
partial projectors come from the oracle; the callback-summed partials equal the one-rank
projector (right and left blocks)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import ctypes

    import oracle
    import synth
    from paper_1404_2891_b200.feast import make_allreduce_callback
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = synth.make_pencil("C2", n=72, m0=6)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    j0, j1 = synth.node_owner_range(len(z), rank, world)
    # this rank's partial right and left blocks, packed [Q | QL] column-major (ld = n) as the
    # library's staging block, then summed in place by the callback (count = float64 values)
    Qr = oracle.project(P.A, P.B, P.X0, z, w, j0, j1)
    Ql = oracle.project(P.A, P.B, P.X0, z, w, j0, j1, left=True)
    buf = np.asfortranarray(np.concatenate([Qr, Ql], axis=1))
    cb = make_allreduce_callback("cpu")
    rc = cb(buf.ctypes.data_as(ctypes.c_void_p).value, 2 * buf.size, None, None)
    assert rc == 0
    # the residual-norm sum: an m-vector of float64
    v = np.full(P.m0, float(rank + 1))
    assert cb(v.ctypes.data_as(ctypes.c_void_p).value, v.size, None, None) == 0
    assert np.all(v == world * (world + 1) / 2)
    # max-over-ranks timing reduction used by bench.py
    import torch
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(out, buf)
        assert t.item() == float(world)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_node_sum_through_callback(tmp_path, world):
    import oracle
    import synth
    out = str(tmp_path / "q.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    P = synth.make_pencil("C2", n=72, m0=6)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    full_r = oracle.project(P.A, P.B, P.X0, z, w)
    full_l = oracle.project(P.A, P.B, P.X0, z, w, left=True)
    got = np.load(out)
    m = P.m0
    assert np.linalg.norm(got[:, :m] - full_r) / np.linalg.norm(full_r) < 1e-13
    assert np.linalg.norm(got[:, m:] - full_l) / np.linalg.norm(full_l) < 1e-13


def test_callback_reports_failure():
    """Without a process group the callback returns nonzero (the library maps it to FEAST_E_COMM)."""
    import ctypes
    from paper_1404_2891_b200.feast import make_allreduce_callback
    v = np.zeros(4)
    assert make_allreduce_callback("cpu")(v.ctypes.data_as(ctypes.c_void_p).value, 4, None, None) == 1
