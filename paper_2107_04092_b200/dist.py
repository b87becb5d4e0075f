"""Multi-GPU plumbing (torch.distributed): the ncclUniqueId the library's
communicator is created from, broadcast from rank 0.
The spike exchange itself is done by libsnn.so (ncclAllGather on the
simulation stream); torch.distributed only bootstraps it."""
from __future__ import annotations


def nccl_unique_id(group=None) -> bytes:
    """128-byte ncclUniqueId created on rank 0 and broadcast to all ranks."""
    import torch
    import torch.distributed as dist
    obj = [None]
    if dist.get_rank(group) == 0:
        obj[0] = bytes(torch.cuda.nccl.unique_id())
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad ncclUniqueId")
    return bytes(uid)


def partitions(n_targets: int, slice_width: int, world: int):
    """All ranks' target ranges (host helper of the C ABI)."""
    from .snn import snn_partition
    return [snn_partition(n_targets, slice_width, world, r) for r in range(world)]
