"""Multi-process bootstrap (plumbing): one process per GPU, torch.distributed for the
handshake only. Every rank exports the CUDA-IPC handle of its symmetric heap, the handles
are all-gathered as bytes, and each rank maps its peers' heaps (seqplan_isp_open_peers).
After this, every collective of the block is a peer-memory kernel of libseqplan_isp.so."""
from __future__ import annotations


def exchange_handles(handle: bytes, world: int, group=None) -> list:
    import torch.distributed as dist
    if world == 1:
        return [handle]
    out = [None] * world
    dist.all_gather_object(out, handle, group=group)
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != len(handle) for h in out):
        raise RuntimeError("peer handle exchange returned malformed handles")
    return [bytes(h) for h in out]


def bootstrap_peers(blk, world: int, group=None) -> None:
    """Maps the peers' heaps into `blk` (an IspBlock). No-op at world == 1."""
    if world == 1:
        return
    import torch.distributed as dist
    handles = exchange_handles(blk.ipc_handle(), world, group)
    blk.open_peers(handles)
    dist.barrier(group=group)
