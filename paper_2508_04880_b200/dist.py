"""Multi-GPU replica mode: one process per GPU, contiguous DFS leaf ranges balanced
by the library's host cost model (tusq_tree_partition), one state vector per GPU, and a single
reduction of the disjoint shot slots.  PAPER.md P:316 ("traverse multiple sub-trees in parallel";
each rank recomputes its prefix instead of receiving a state copy, reading #20).

The slot arrays are disjoint across ranks, so the SUM all-reduce is exact and the result is
bit-identical for any number of ranks (shot streams are keyed by leaf id)."""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def leaf_range(tree, rank: int, world: int, precision: int = 128):
    b = tree.partition(world, precision)
    return int(b[rank]), int(b[rank + 1])


def tree_digest(tree) -> int:
    """64-bit digest of the canonical tree bytes (every rank must build the identical tree)."""
    import hashlib
    return int.from_bytes(hashlib.sha256(tree.serialize()).digest()[:8], "little") & ((1 << 63) - 1)


def run_tree_distributed(tree, precision: int = 128, d_state=None, stream=None, flags: int = 0,
                         group=None, run_range: Optional[Callable[[int, int], np.ndarray]] = None,
                         device: str = "cuda"):
    """Run this rank's leaf range and sum the slot arrays over the process group.

    run_range(leaf_begin, leaf_end) -> u64[S] slots (zeros outside the range); defaults to the
    CUDA path (tusq_run_tree).  Returns (slots u64[S], (leaf_begin, leaf_end))."""
    import torch
    import torch.distributed as dist

    rank, world = (dist.get_rank(group), dist.get_world_size(group)) if dist.is_initialized() else (0, 1)
    lb, le = leaf_range(tree, rank, world, precision)
    if world > 1:
        d = torch.tensor([tree_digest(tree)], dtype=torch.int64, device=device)
        allg = [torch.zeros_like(d) for _ in range(world)]
        dist.all_gather(allg, d, group=group)
        if any(int(x.item()) != int(d.item()) for x in allg):
            raise RuntimeError("ranks built different trees (seed or inputs differ)")
    if run_range is None:
        from . import tusq as T

        def run_range(b, e):
            out = np.zeros(tree.info()["S1"], dtype=np.uint64)
            if e > b:
                T.run_tree(tree, precision, d_state=d_state, stream=stream, leaf_begin=b, leaf_end=e,
                           flags=flags, out_slots=out)
            return out
    slots = run_range(lb, le)
    if world > 1:
        t = torch.from_numpy(slots.view(np.int64).copy()).to(device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        slots = t.cpu().numpy().view(np.uint64)
    return slots, (lb, le)


def share_unique_id(group=None, unique_id: Optional[Callable[[], bytes]] = None) -> bytes:
    """Rank 0 draws the NCCL unique id (tusq_comm_unique_id); every rank receives it over the group."""
    import torch.distributed as dist

    from . import tusq as T

    box = [(unique_id or T.Comm.unique_id)()] if dist.get_rank(group) == 0 else [None]
    dist.broadcast_object_list(box, src=0, group=group)
    if not isinstance(box[0], (bytes, bytearray)) or len(box[0]) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(box[0])


def make_comm(device: int, group=None, unique_id: Optional[Callable[[], bytes]] = None):
    """One tusq_comm per rank of the torch.distributed group, joined to the library's own NCCL
    communicator (tusq_comm_init): the sharded mode's exchanges and the replica
    mode's slot reduction (tusq_reduce_slots / exec.comm).  Returns (comm, uid bytes)."""
    import torch.distributed as dist

    from . import tusq as T

    uid = share_unique_id(group, unique_id)
    return T.Comm.nccl(uid, dist.get_world_size(group), dist.get_rank(group), device), uid


make_sharded_comm = make_comm
