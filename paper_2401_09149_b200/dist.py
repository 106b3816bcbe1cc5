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
    """Maps the peers' heaps into `blk` (an IspBlock), then sets up the NVLink SHARP reduce-scatter
    where it applies (bootstrap_nvls). No-op at world == 1."""
    if world == 1:
        return
    import torch.distributed as dist
    handles = exchange_handles(blk.ipc_handle(), world, group)
    blk.open_peers(handles)
    dist.barrier(group=group)
    bootstrap_nvls(blk, world, group)


def bootstrap_nvls(blk, world: int, group=None) -> bool:
    """NVLink SHARP reduce-scatter buffers (seqplan_isp_nvls_*): rank 0 creates the multicast
    object and publishes (pid, fd) of its exported POSIX handle; every rank attaches (the others
    duplicate the fd out of rank 0's process) and adds its GPU; after a barrier every rank binds
    and maps its memory. Every rank follows rank 0's decision, and a failure anywhere releases it
    everywhere (the push reduce-scatter is used). Returns whether the block uses NVLS."""
    if world == 1 or not hasattr(blk, "nvls_export"):
        return False
    import torch.distributed as dist
    rank = dist.get_rank(group)
    src = dist.get_global_rank(group, 0) if group is not None else 0
    # one multicast object spans distinct GPUs: ranks sharing a GPU (an oversubscribed box) keep
    # the push reduce-scatter
    import os
    import socket
    where = [None] * world
    dist.all_gather_object(where, (socket.gethostname(), os.environ.get("CUDA_VISIBLE_DEVICES"),
                                   getattr(blk, "device", None)), group=group)
    if len(set(where)) != world:
        return False
    info = [blk.nvls_export() if rank == 0 else None]
    dist.broadcast_object_list(info, src=src, group=group)
    if info[0] is None:
        return False

    def agree(ok: bool) -> bool:
        oks = [None] * world
        dist.all_gather_object(oks, bool(ok), group=group)
        return all(oks)

    ok = blk.nvls_attach(*(info[0] if rank != 0 else (0, -1)))
    if agree(ok):
        dist.barrier(group=group)
        if agree(blk.nvls_bind()):
            dist.barrier(group=group)
            return True
    blk.nvls_release()
    dist.barrier(group=group)
    return False
