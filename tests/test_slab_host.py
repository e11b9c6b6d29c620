"""Host-side logic of z-slab sharding, on CPU: the partition and the NCCL
bootstrap (unique id broadcast over a world-size-2 gloo group, as bench.py does
under torchrun)."""
import os
import socket

import numpy as np
import pytest


def test_slab_partition(mssz):
    for Z in (4, 5, 17, 48, 1024):
        for p in range(1, min(Z // 2, 64) + 1):
            rows = [mssz.slab_range(Z, p, r) for r in range(p)]
            assert rows[0][0] == 0 and rows[-1][1] == Z
            for r, (z0, z1, wz0, wz1) in enumerate(rows):
                assert z1 - z0 >= 2
                assert wz0 == max(0, z0 - 2) and wz1 == min(Z, z1 + 2)
                if r:
                    assert rows[r - 1][1] == z0
    with pytest.raises(mssz.Error) as e:
        mssz.slab_range(5, 3, 0)
    assert e.value.kind() == mssz.ErrKind.usage
    with pytest.raises(mssz.Error):
        mssz.slab_range(100, 2, 2)


def test_unique_id_and_no_gpu(mssz):
    uid = mssz.SlabComm.unique_id()
    assert len(uid) == 128 and any(uid)
    if mssz.library().mssz_cu_device_count() == 0:
        with pytest.raises(mssz.Error) as e:  # no CPU fallback
            mssz.SlabComm(uid, 1, 0, 0)
        assert e.value.kind() == mssz.ErrKind.cuda


def _worker(rank, world, port, out):
    import torch.distributed as dist
    import paper_2406_09423_b200 as P
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    obj = [P.SlabComm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    z0, z1, wz0, wz1 = P.slab_range(64, world, rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, (obj[0], z0, z1))
    dist.destroy_process_group()
    out.put((rank, gathered))


def test_gloo_bootstrap_world2(mssz):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        ids = {g[0] for g in res[r]}
        assert len(ids) == 1  # every rank holds rank 0's id
        spans = sorted((g[1], g[2]) for g in res[r])
        assert spans == [(0, 32), (32, 64)]
