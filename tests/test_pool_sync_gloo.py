"""Multi-rank pool synchronisation on CPU: two
processes over gloo all-gather fixed-size best records (libfg host code packs and
merges them) and must agree on the same deterministic minimum (R20)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from golden_io import load_scheme


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_20317_b200 import fg
        from paper_2511_20317_b200.pool_sync import PoolSync, merge_gathered
        from oracle import Oracle
        orc = Oracle()
        R = 32
        _, _, _, strassen = load_scheme("sec36_after.txt")
        before = load_scheme("sec36_before.txt")[3]
        naive = orc.naive(2, 2, 2)
        # rank 0 holds the naive scheme (rank 8); rank 1 holds two rank-7 schemes of
        # equal additions: the lower global walker id must win everywhere
        if rank == 0:
            rec = fg.fg_record_pack(2, 2, 2, 0, R, naive, 3)
        else:
            rec = fg.fg_record_pack(2, 2, 2, 0, R, strassen, 17)
        sync = PoolSync(graph=None, world=world)
        recs = sync.gather_records(rec)
        res = merge_gathered(recs, world, R)
        # second round: rank 0 now reports the un-normalised variant with id 9
        rec2 = fg.fg_record_pack(2, 2, 2, 0, R, orc.normalize(2, 2, 2, before), 9) if rank == 0 else rec
        res2 = merge_gathered(sync.gather_records(rec2), world, R)
        q.put((rank, res["rank"], res["additions"], res["walker_id"], res["coeffs"].tobytes(),
               res2["rank"], res2["walker_id"]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_pool_sync():
    from paper_2511_20317_b200.build import build_libfg
    build_libfg()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    _, _, _, strassen = load_scheme("sec36_after.txt")
    for (rank, rk, adds, wid, cb, rk2, wid2) in out:
        assert (rk, adds, wid) == (7, 18, 17)
        assert np.frombuffer(cb, np.int8).reshape(7, -1).tolist() == strassen.tolist()
        assert (rk2, wid2) == (7, 9)          # same rank and additions, lower id wins
    assert out[0][1:] == out[1][1:]
