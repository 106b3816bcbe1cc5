"""Worker for tests/test_coresident_gpu.py (run in a subprocess with CUDA_MODULE_LOADING=EAGER:
under lazy loading the first launch of a kernel waits for the device to go idle, which co-resident
ranks waiting for each other on the device never do). Prints one JSON line."""
import json
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from oracle import block as ob  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402

H, D, S = 1024, 8, 1024


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def inputs():
    sh = ob.Shape(H=H, D=D, S=S)
    w = ob.make_weights(sh)
    x = torch.from_numpy(ob.make_activation(sh, ob.TID_X)).bfloat16()
    dy = torch.from_numpy(ob.make_activation(sh, ob.TID_DY)).bfloat16()
    return sh, w, x, dy


def make_ranks(p, w, flags=0):
    blocks = [capi.IspBlock(H, D, S, world=p, rank=r, device=0, flags=flags) for r in range(p)]
    capi.link_local_peers(blocks)
    for r, b in enumerate(blocks):
        for t in range(7):
            flat = w[t].reshape(-1)
            per = flat.size // p
            b.set_weight_shard(t, flat[r * per:(r + 1) * per])
    return blocks


def run_steps(blocks, xs, dys, ys, dxs, streams, steps, adamw, lr=1e-3):
    """Each rank issues its own sequence (steps x fwd, bwd, AdamW after every step but the last)
    from its own host thread, as one process per GPU would; the ranks meet on the device only."""
    errors = []

    def rank_loop(b, x, y, dy, dx, s):
        try:
            for k in range(steps):
                b.fwd(x, y, s)
                b.bwd(dy, dx, s)
                if adamw and k + 1 < steps:
                    b.adamw_step(lr, k + 1, stream=s)
        except Exception as ex:  # noqa: BLE001
            errors.append(repr(ex))

    th = [threading.Thread(target=rank_loop, args=a, daemon=True) for a in zip(blocks, xs, ys, dys, dxs, streams)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    if any(t.is_alive() for t in th):
        print(json.dumps({"error": "a rank did not finish issuing (device deadlock)"}), flush=True)
        sys.exit(3)
    if errors:
        raise RuntimeError(errors)


def setup(p, flags=0):
    dev = torch.device("cuda", 0)
    sh, w, x, dy = inputs()
    blocks = make_ranks(p, w, flags)
    T = S // p
    xs = [x[r * T:(r + 1) * T].to(dev) for r in range(p)]
    dys = [dy[r * T:(r + 1) * T].to(dev) for r in range(p)]
    ys = [torch.empty_like(t) for t in xs]
    dxs = [torch.empty_like(t) for t in xs]
    streams = [torch.cuda.Stream() for _ in range(p)]
    torch.cuda.synchronize()
    return sh, w, x, dy, blocks, xs, dys, ys, dxs, streams


def parity(p, adamw):
    sh, w, x, dy, blocks, xs, dys, ys, dxs, streams = setup(p)
    run_steps(blocks, xs, dys, ys, dxs, streams, 3, adamw)
    torch.cuda.synchronize()
    # the last step vs the oracle at the weights it ran on (the fp32 masters after the updates)
    ws = [np.concatenate([b.weight_shard(t) for b in blocks]).reshape(s) for t, s in enumerate(sh.weight_shapes())]
    res = {"moved": float(min(np.abs(a - b).max() for a, b in zip(ws, w)))}
    y_ref, dx_ref, g_ref = ob.block(sh, ws, x.float().numpy(), dy.float().numpy(), p=1)
    res["y"] = rel(torch.cat(ys).float().cpu(), y_ref)
    res["dx"] = rel(torch.cat(dxs).float().cpu(), dx_ref)
    for t in range(7):
        res[capi.W_NAMES[t]] = rel(np.concatenate([b.grad_shard(t) for b in blocks]), g_ref[t].reshape(-1))
    res["push"] = [int(v) for v in (0,)]
    for b in blocks:
        b.close()
    return res


def timelines(p):
    sh, w, x, dy, blocks, xs, dys, ys, dxs, streams = setup(p, capi.FLAG_TIMELINE)
    run_steps(blocks, xs, dys, ys, dxs, streams, 1, False)  # warm-up: pools, gathers primed
    for b in blocks:
        b.timeline()
    run_steps(blocks, xs, dys, ys, dxs, streams, 1, False)
    out = [b.timeline() for b in blocks]
    for b in blocks:
        b.close()
    return {"timelines": out}


if __name__ == "__main__":
    mode, p = sys.argv[1], int(sys.argv[2])
    if mode == "parity":
        r = parity(p, sys.argv[3] == "adamw")
    else:
        r = timelines(p)
    print("RESULT " + json.dumps(r), flush=True)
