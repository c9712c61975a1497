"""The pool synchronisation's NCCL branch on the device.
Only one GPU is available to the tests, so this runs a 1-rank NCCL process group: the
record all-gather goes through NCCL on cuda:0 (all_gather_into_tensor) and the merge
through libfg; the 2-rank merge logic is covered over gloo in test_pool_sync_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2511_20317_b200 import fg
        from paper_2511_20317_b200.pool_sync import PoolSync
        from paper_2511_20317_b200.inputs import WORKLOADS
        wl = WORKLOADS["c2_333_zt"]
        g = fg.FlipGraph(wl.m, wl.n, wl.p, wl.ring, wl.r_cap, 512, 0, 0, torch.cuda.current_stream().cuda_stream)
        g.seed_naive()
        g.walk(3000, wl.seed)
        local = g.best()
        sync = PoolSync(g)
        assert dist.get_backend() == "nccl" and sync.world == 1
        rec = g.export_best()
        got = sync.gather_records(rec)                  # NCCL all-gather on cuda:0
        merged = sync.exchange()                        # export, all-gather, import (libfg)
        q.put(("ok", bool(np.array_equal(got.reshape(-1), rec)), local["rank"], local["additions"],
               merged["rank"], merged["additions"], bool(np.array_equal(local["coeffs"], merged["coeffs"]))))
        g.close()
    except Exception as e:  # noqa: BLE001
        q.put(("error", repr(e)))
    finally:
        dist.destroy_process_group()


def test_nccl_record_exchange_one_rank():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert res[0] == "ok", res
    _, same, lr, la, mr, ma, same_rows = res
    assert same and (lr, la) == (mr, ma) and same_rows
