"""Host logic of the column-sharded path on the CPU: the layout exported by the
C ABI (randutv_dist_layout, no GPU needed) and the Python sharding helpers,
exercised by a world_size-2 torch.distributed job over gloo (127.0.0.1):
every rank shards a seeded global matrix with the library's layout, the shards
are exchanged, and the reassembly must reproduce the matrix bit for bit."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def built():
    from paper_2002_06960_b200 import build as b
    b.build()


@pytest.mark.parametrize("m,n,b,P", [(1000, 700, 64, 1), (1000, 700, 64, 3), (96, 96, 32, 4), (65536, 65536, 512, 8),
                                     (262144, 8192, 256, 8), (50, 50, 100, 2)])
def test_layout_partitions(built, m, n, b, P):
    from paper_2002_06960_b200.randutv import dist_layout, local_columns
    cols, urows, vrows = [], [], []
    for p in range(P):
        lay = dist_layout(m, n, b, P, p)
        lc = local_columns(n, b, P, p)
        assert lay["ncols"] == len(lc)
        cols.extend(lc.tolist())
        urows.extend(range(lay["u0"], lay["u1"]))
        vrows.extend(range(lay["v0"], lay["v1"]))
        # block-cyclic: every local column block is a whole global block owned by p
        bb = min(b, n)
        assert all((c // bb) % P == p for c in lc)
    assert sorted(cols) == list(range(n))
    assert urows == list(range(m)) and vrows == list(range(n))


def test_layout_errors(built):
    import ctypes
    from paper_2002_06960_b200.randutv import load_library
    lib = load_library()
    out = (ctypes.c_int64 * 5)()
    assert lib.randutv_dist_layout(10, 20, 4, 2, 0, out) == -1
    assert lib.randutv_dist_layout(10, 10, 0, 2, 0, out) == -3
    assert lib.randutv_dist_layout(10, 10, 4, 2, 2, out) == -5


def _worker(rank, world, port, m, n, b, q_out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2002_06960_b200.randutv import dist_layout, local_columns
        A = np.asfortranarray(np.random.default_rng(42).standard_normal((m, n)))
        lc = local_columns(n, b, world, rank)
        lay = dist_layout(m, n, b, world, rank)
        shard = {"cols": lc, "A": A[:, lc], "u": (lay["u0"], lay["u1"]), "v": (lay["v0"], lay["v1"])}
        allshards = [None] * world
        dist.all_gather_object(allshards, shard)
        R = np.zeros_like(A)
        for s in allshards:
            R[:, s["cols"]] = s["A"]
        ok = np.array_equal(R, A)
        ok &= sum(s["u"][1] - s["u"][0] for s in allshards) == m
        ok &= sum(s["v"][1] - s["v"][0] for s in allshards) == n
        # the NCCL-id bootstrap path: rank 0's bytes reach every rank unchanged
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ok &= obj[0] == bytes(range(128))
        q_out.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_roundtrip(built):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 300, 250, 32, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
