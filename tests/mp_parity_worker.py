"""torchrun worker: multi-process ISP block (real CUDA IPC peers) vs the CPU oracle.
Launched by tests/test_multiprocess_gpu.py; prints one JSON line per rank."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import block as ob  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402
from paper_2401_09149_b200.dist import bootstrap_peers  # noqa: E402


def _device(rank):
    """This rank's GPU and the bootstrap group. MP_RANKS_PER_GPU > 1 oversubscribes the box (e.g.
    8 ranks on 4 GPUs): rank r uses GPU r % count, and the bootstrap runs over gloo (NCCL refuses
    two ranks on one device); the block's own transport is CUDA IPC either way."""
    local = int(os.environ.get("LOCAL_RANK", rank))
    over = int(os.environ.get("MP_RANKS_PER_GPU", "1")) > 1
    if over:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if over:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    return local, dev


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def steps_mode(H, D, S, adamw):
    """Production-path check (no flags, no host synchronisation inside): 3 back-to-back fwd/bwd
    steps on one stream, optionally with an AdamW update of the shards after each, as a training
    loop issues them; cross-step reuse of the peer exchange buffers then rests on the in-step
    barriers alone. Step 3's y / dx / gradient shards and the final weight shards vs the oracle
    running the same sequence."""
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local, dev = _device(rank)
    sh = ob.Shape(H=H, D=D, S=S)
    w = ob.make_weights(sh)
    x = torch.from_numpy(ob.make_activation(sh, ob.TID_X)).bfloat16()
    dy = torch.from_numpy(ob.make_activation(sh, ob.TID_DY)).bfloat16()
    T = S // world
    blk = capi.IspBlock(H, D, S, world=world, rank=rank, device=local, flags=0)
    bootstrap_peers(blk, world)
    for t in range(7):
        flat = w[t].reshape(-1)
        per = flat.size // world
        blk.set_weight_shard(t, flat[rank * per:(rank + 1) * per])
    dist.barrier()
    xd = x[rank * T:(rank + 1) * T].to(dev)
    dyd = dy[rank * T:(rank + 1) * T].to(dev)
    y, dx = torch.empty_like(xd), torch.empty_like(xd)
    lr = 1e-3
    w0 = [blk.weight_shard(t) for t in range(7)]
    for k in range(3):  # AdamW after steps 1 and 2: step 3 runs on twice-updated weights
        blk.fwd(xd, y)
        blk.bwd(dyd, dx)
        if adamw and k < 2:
            blk.adamw_step(lr, k + 1)
    torch.cuda.synchronize()
    res = {"rank": rank}
    # step 3 vs the oracle at the weights the device used in step 3 (its fp32 masters); the
    # update rule itself is checked element-wise in test_adamw_step_matches_oracle
    shards = [blk.weight_shard(t) for t in range(7)]
    moved = [float(np.abs(a - b).max()) for a, b in zip(shards, w0)]
    allw = [None] * world
    dist.all_gather_object(allw, shards)
    if rank == 0:
        ws = [np.concatenate([allw[q][t] for q in range(world)]).reshape(s) for t, s in
              enumerate(sh.weight_shapes())]
        y_ref, dx_ref, g_ref = ob.block(sh, ws, x.float().numpy(), dy.float().numpy(), p=1)
        ref = (y_ref, dx_ref, [g.reshape(-1) for g in g_ref])
    else:
        ref = None
    obj = [ref]
    dist.broadcast_object_list(obj, src=0)
    y_ref, dx_ref, g_ref = obj[0]
    res["y"] = rel(y.float().cpu(), y_ref[rank * T:(rank + 1) * T])
    res["dx"] = rel(dx.float().cpu(), dx_ref[rank * T:(rank + 1) * T])
    for t in range(7):
        per = g_ref[t].size // world
        res[capi.W_NAMES[t]] = rel(blk.grad_shard(t), g_ref[t][rank * per:(rank + 1) * per])
        if adamw:  # the updates happened (0 = moved)
            res["w_" + capi.W_NAMES[t] + "_static"] = float(moved[t] == 0.0)
    print(json.dumps(res), flush=True)
    blk.close()
    dist.barrier()
    dist.destroy_process_group()


def main():
    H, D, S = (int(v) for v in sys.argv[1:4])
    if len(sys.argv) > 4 and sys.argv[4] in ("steps", "steps_adamw"):
        steps_mode(H, D, S, sys.argv[4] == "steps_adamw")
        return
    fused = len(sys.argv) > 4 and sys.argv[4] == "fused"
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local, dev = _device(rank)
    sh = ob.Shape(H=H, D=D, S=S)
    w = ob.make_weights(sh)
    x = torch.from_numpy(ob.make_activation(sh, ob.TID_X)).bfloat16()
    dy = torch.from_numpy(ob.make_activation(sh, ob.TID_DY)).bfloat16()
    T = S // world
    flags = capi.FLAG_TIMELINE | (capi.FLAG_FUSED_BWD if fused else 0)
    blk = capi.IspBlock(H, D, S, world=world, rank=rank, device=local, flags=flags)
    bootstrap_peers(blk, world)
    for t in range(7):
        flat = w[t].reshape(-1)
        per = flat.size // world
        blk.set_weight_shard(t, flat[rank * per:(rank + 1) * per])
    dist.barrier()
    xd = x[rank * T:(rank + 1) * T].to(dev)
    dyd = dy[rank * T:(rank + 1) * T].to(dev)
    y, dx = torch.empty_like(xd), torch.empty_like(xd)
    for _ in range(2):  # second step checks recycling / epochs
        blk.fwd(xd, y)
        blk.bwd(dyd, dx)
        torch.cuda.synchronize()
    res = {"rank": rank}
    if rank == 0:
        y_ref, dx_ref, g_ref = ob.block(sh, w, x.float().numpy(), dy.float().numpy(), p=1)
        ref = (y_ref, dx_ref, g_ref)
    else:
        ref = None
    obj = [ref]
    dist.broadcast_object_list(obj, src=0)
    y_ref, dx_ref, g_ref = obj[0]
    res["y"] = rel(y.float().cpu(), y_ref[rank * T:(rank + 1) * T])
    res["dx"] = rel(dx.float().cpu(), dx_ref[rank * T:(rank + 1) * T])
    for t in range(7):
        flat = g_ref[t].reshape(-1)
        per = flat.size // world
        res[capi.W_NAMES[t]] = rel(blk.grad_shard(t), flat[rank * per:(rank + 1) * per])
    res["timeline_events"] = len(blk.timeline())
    if os.environ.get("MP_REPORT_NVLS"):
        res["nvls_active"] = blk.nvls_active()
    print(json.dumps(res), flush=True)
    blk.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
