"""Population synchronisation across GPUs.

Walkers shard by global id (rank r owns ids [r*W, (r+1)*W)); the Philox counter
uses the global id, so trajectories do not depend on the GPU count.  Between walk
phases each rank exports one fixed-size best record (fg_export_best), the records
are all-gathered (torch.distributed: NCCL over NVLink on GPUs, gloo on CPU), and
every rank merges them with the same deterministic rule (R20, fg_import_best).
The merge itself runs in libfg (host C++); this module only moves bytes.
"""
from __future__ import annotations

import numpy as np


class PoolSync:
    def __init__(self, graph, world: int | None = None, group=None):
        import torch.distributed as dist
        self.g = graph
        self.group = group
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.world = world

    def gather_records(self, rec: np.ndarray) -> np.ndarray:
        """All-gather one uint8 record per rank; returns world x bytes."""
        import torch
        import torch.distributed as dist
        if self.world == 1 and not dist.is_initialized():
            return rec.reshape(1, -1)
        backend = dist.get_backend(self.group)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        t = torch.from_numpy(rec).to(dev)
        out = torch.empty(self.world * rec.size, dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy().reshape(self.world, -1)

    def exchange(self) -> dict:
        """Export the local best, all-gather, merge into the pool; returns the
        box-wide best (rank, additions, walker id, coeffs)."""
        import torch.distributed as dist
        if self.world > 1 or dist.is_initialized():
            recs = self.gather_records(self.g.export_best())
            self.g.import_best(np.ascontiguousarray(recs.reshape(-1)), self.world)
        return self.g.best()


def merge_gathered(records: np.ndarray, world: int, r_cap: int) -> dict:
    """Host-only merge of all-gathered records (for tests and tools)."""
    from . import fg
    out = fg.fg_record_merge(np.ascontiguousarray(records.reshape(-1)), world)
    return fg.fg_record_unpack(out, r_cap)
