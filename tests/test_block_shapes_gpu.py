"""Block parity at the B200 BASELINE shapes (BASELINE.json configs 2-5): the sm_100a ISP block
through the C ABI vs an fp32 PyTorch restatement run on the GPU (tests/reference_torch.py, itself
pinned to the CPU oracle by tests/test_oracle.py), on identical inputs: x, dy and the weights as
the device holds them (bf16 working shards of the fp32 masters), computed in fp32 from there.

Bar (BASELINE.json north_star): rel-L2 <= 1e-2 for bf16 activations and gradients. p = 1 runs one
context; p > 1 runs the group mode (p ranks on one GPU, the multi-process kernels with the peers'
buffers on the same device); weight-gradient shards are compared per rank (ShardingLayout E/F).
"""
import numpy as np
import pytest
import torch

from oracle import block as ob
from paper_2401_09149_b200 import capi
from tests import reference_torch as rt

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


_CACHE = {}


def reference(H, D, S, dev):
    key = (H, D, S)
    if key not in _CACHE:
        _CACHE.clear()
        torch.cuda.empty_cache()
        sh = ob.Shape(H=H, D=D, S=S)
        w = ob.make_weights(sh)
        x = torch.from_numpy(ob.make_activation(sh, ob.TID_X)).bfloat16()
        dy = torch.from_numpy(ob.make_activation(sh, ob.TID_DY)).bfloat16()
        W = [torch.from_numpy(t).to(dev).bfloat16().float() for t in w]  # the bf16 working weights
        y, dx, g = rt.block_fwd_bwd(x.float().to(dev), dy.float().to(dev), W, D)
        _CACHE[key] = (w, x, dy, y, dx, [t.reshape(-1) for t in g])
        del W
        torch.cuda.empty_cache()
    return _CACHE[key]


def load_weights(blk, w, p, r):
    for t in range(7):
        flat = w[t].reshape(-1)
        per = flat.size // p
        blk.set_weight_shard(t, flat[r * per:(r + 1) * per])


@pytest.mark.parametrize("H,D,S,p", [
    (4096, 32, 4096, 1), (4096, 32, 4096, 2), (4096, 32, 4096, 4), (4096, 32, 4096, 8),  # 7B, S = 4K
    (4096, 32, 2048, 8),                                                                  # 7B, S = 2K
    (5120, 40, 2048, 1), (5120, 40, 2048, 8),                                             # 20B block (40 heads)
])
def test_block_at_baseline_shape(cuda, H, D, S, p):
    torch.backends.cuda.matmul.allow_tf32 = False
    w, x, dy, y_ref, dx_ref, g_ref = reference(H, D, S, cuda)
    T = S // p
    if p == 1:
        blk = capi.IspBlock(H, D, S, world=1)
        blocks = [blk]
        load_weights(blk, w, 1, 0)
        xs, dys = [x.to(cuda)], [dy.to(cuda)]
        ys, dxs = [torch.empty_like(xs[0])], [torch.empty_like(xs[0])]
        blk.fwd(xs[0], ys[0])
        blk.bwd(dys[0], dxs[0])
    else:
        grp = capi.IspGroup(H, D, S, world=p)
        blocks = [grp.rank(r) for r in range(p)]
        for r, b in enumerate(blocks):
            load_weights(b, w, p, r)
        xs = [x[r * T:(r + 1) * T].to(cuda) for r in range(p)]
        dys = [dy[r * T:(r + 1) * T].to(cuda) for r in range(p)]
        ys = [torch.empty_like(t) for t in xs]
        dxs = [torch.empty_like(t) for t in xs]
        grp.fwd(xs, ys)
        grp.bwd(dys, dxs)
    torch.cuda.synchronize()
    errs = {"y": rel(torch.cat(ys).float(), y_ref), "dx": rel(torch.cat(dxs).float(), dx_ref)}
    for t in range(7):
        got = torch.from_numpy(np.concatenate([b.grad_shard(t) for b in blocks])).to(cuda)
        errs[capi.W_NAMES[t]] = rel(got, g_ref[t])
    (grp.close() if p > 1 else blk.close())
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, (errs, bad)
