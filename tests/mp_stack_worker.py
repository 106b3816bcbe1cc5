"""torchrun worker: multi-process 2-layer ISP stack (real CUDA IPC peers, inter-layer prefetch on
one comm stream) vs the CPU oracle block chained twice. Launched by tests/test_multiprocess_gpu.py;
prints one JSON line per rank."""
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


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def main():
    H, D, S, L = (int(v) for v in sys.argv[1:5])
    recompute = len(sys.argv) > 5 and sys.argv[5] == "recompute"
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    sh = ob.Shape(H=H, D=D, S=S)
    ws = [ob.make_weights(sh, seed=ob.SEED + l) for l in range(L)]
    x = torch.from_numpy(ob.make_activation(sh, ob.TID_X)).bfloat16()
    dy = torch.from_numpy(ob.make_activation(sh, ob.TID_DY)).bfloat16()
    T = S // world
    pol = capi.make_policy(consolidate=2) if recompute else None
    st = capi.IspStack(L, H, D, S, world=world, rank=rank, device=local, flags=capi.FLAG_TIMELINE,
                       recompute=recompute, policy=pol)
    for l in range(L):
        blk = st.layer(l)
        bootstrap_peers(blk, world)
        for t in range(7):
            flat = ws[l][t].reshape(-1)
            per = flat.size // world
            blk.set_weight_shard(t, flat[rank * per:(rank + 1) * per])
    dist.barrier()
    xd = x[rank * T:(rank + 1) * T].to(dev)
    dyd = dy[rank * T:(rank + 1) * T].to(dev)
    y, dx = torch.empty_like(xd), torch.empty_like(xd)
    for _ in range(2):  # second step checks recycling / epochs
        st.fwd(xd, y)
        st.bwd(dyd, dx)
        torch.cuda.synchronize()
    ref = None
    if rank == 0:  # oracle chain with the GPU's bf16 rounding at layer boundaries
        xs = [x.float().numpy()]
        for l in range(L):
            yl, _, _ = ob.block(sh, ws[l], xs[-1], np.zeros_like(xs[-1]), p=1)
            xs.append(bf16(yl))
        g_in, grads = dy.float().numpy(), [None] * L
        for l in reversed(range(L)):
            _, dxl, g = ob.block(sh, ws[l], xs[l], g_in, p=1)
            grads[l] = g
            g_in = bf16(dxl)
        ref = (yl, dxl, grads)
    obj = [ref]
    dist.broadcast_object_list(obj, src=0)
    y_ref, dx_ref, g_ref = obj[0]
    res = {"rank": rank, "y": rel(y.float().cpu(), y_ref[rank * T:(rank + 1) * T]),
           "dx": rel(dx.float().cpu(), dx_ref[rank * T:(rank + 1) * T])}
    for l in range(L):
        for t in range(7):
            flat = g_ref[l][t].reshape(-1)
            per = flat.size // world
            res[f"L{l}_{capi.W_NAMES[t]}"] = rel(st.layer(l).grad_shard(t), flat[rank * per:(rank + 1) * per])
    print(json.dumps(res), flush=True)
    st.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
