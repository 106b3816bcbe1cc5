"""Pins the CPU fp32 oracle (oracle/block_oracle.c).

The reference computes no tensors, so numeric parity is "unpinned" by it
(SURVEY.md §8c). The oracle is pinned instead by (1) an independent PyTorch-autograd
restatement of the same block, (2) the ISP-sharded simulation agreeing with the
unsharded block to rel-L2 <= 1e-5 (BASELINE.json fp32 tolerance), and (3) frozen
values of the index-keyed generator.
"""
import numpy as np
import pytest
import torch

from oracle import block as ob
from tests import reference_torch as rt


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


SMALL = ob.Shape(H=256, D=4, S=256)  # d = 64, I = 768


@pytest.fixture(scope="module")
def small_case():
    w = ob.make_weights(SMALL)
    x = ob.make_activation(SMALL, ob.TID_X)
    dy = ob.make_activation(SMALL, ob.TID_DY)
    return w, x, dy, ob.block(SMALL, w, x, dy, p=1)


def test_keyed_generator_frozen_values():
    # splitmix64 -> Box-Muller in double; frozen so drift is caught.
    v = [ob.lib().ob_keyed_normal(ob.SEED, 0, i) for i in range(4)]
    v2 = [ob.lib().ob_keyed_normal(ob.SEED, 3, 1000003 + i) for i in range(2)]
    np.testing.assert_allclose(v + v2, FROZEN, rtol=0, atol=1e-15)


def test_keyed_generator_is_shard_independent():
    full = ob.fill(ob.TID_WQKV, 4096)
    for p in (2, 4, 8):
        per = 4096 // p
        parts = np.concatenate([ob.fill(ob.TID_WQKV, per, offset=r * per) for r in range(p)])
        assert np.array_equal(parts, full)
    z = ob.fill(ob.TID_X, 1 << 18)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


def test_oracle_matches_torch_autograd(small_case):
    w, x, dy, (y, dx, grads) = small_case
    W = [torch.from_numpy(a.copy()).double() for a in w]
    ty, tdx, tg = rt.block_fwd_bwd(torch.from_numpy(x).double(), torch.from_numpy(dy).double(), W,
                                   SMALL.D, SMALL.eps, SMALL.rope_base)
    assert rel(y, ty.numpy()) < 1e-5
    assert rel(dx, tdx.numpy()) < 1e-5
    for g, t in zip(grads, tg):
        assert rel(g, t.numpy()) < 1e-5


@pytest.mark.parametrize("p", [2, 4])
def test_isp_sharded_matches_unsharded_fp32(small_case, p):
    w, x, dy, (y, dx, grads) = small_case
    y2, dx2, g2 = ob.block(SMALL, w, x, dy, p=p)
    assert rel(y2, y) <= 1e-5 and rel(dx2, dx) <= 1e-5
    for a, b in zip(g2, grads):
        assert rel(a, b) <= 1e-5


def test_cpu_ref_config_p2():
    """BASELINE config 1: H=512, 8 heads, S=1K, fp32, simulated 2-way ISP on the host."""
    sh = ob.Shape(H=512, D=8, S=1024)
    w = ob.make_weights(sh)
    x, dy = ob.make_activation(sh, ob.TID_X), ob.make_activation(sh, ob.TID_DY)
    y1, dx1, g1 = ob.block(sh, w, x, dy, p=1)
    y2, dx2, g2 = ob.block(sh, w, x, dy, p=2)
    assert rel(y2, y1) <= 1e-5 and rel(dx2, dx1) <= 1e-5
    assert all(rel(a, b) <= 1e-5 for a, b in zip(g2, g1))


def test_oracle_rejects_bad_sharding():
    with pytest.raises(ValueError):
        ob.block(ob.Shape(H=256, D=4, S=256), ob.make_weights(SMALL), np.zeros((256, 256), np.float32),
                 np.zeros((256, 256), np.float32), p=8)  # 4 heads not divisible by 8


FROZEN = [-1.1993611852119628, -0.059745141150991395, 0.8620070529295685, -0.5620351665735817,
          -0.45045825860339406, 0.16131780976187002]


def test_block_sample_is_the_block_work_of_its_rows():
    """bench.py's bounded CPU sample (ob_block_sample): with every position sampled it is the full
    block (y, dx, grads); with a subset and the true K|V of the prefix, the sampled rows' forward
    outputs equal the full block's rows; its FLOPs are n/S of the block's."""
    sh = ob.Shape(H=256, D=4, S=256)
    w = ob.make_weights(sh)
    x = ob.make_activation(sh, ob.TID_X)
    dy = ob.make_activation(sh, ob.TID_DY)
    y, dx, g = ob.block(sh, w, x, dy)
    kv = np.zeros((sh.S, 2 * sh.H), np.float32)
    dkv = np.zeros_like(kv)
    y2, dx2, g2 = ob.block_sample(sh, w, np.arange(sh.S), x, dy, kv, dkv)
    assert rel(y2, y) < 1e-5 and rel(dx2, dx) < 1e-5
    for a, b in zip(g2, g):
        assert rel(a.reshape(-1), b.reshape(-1)) < 1e-5
    pos = np.arange(8) * 32 + 16
    y3, _, _ = ob.block_sample(sh, w, pos, x[pos], dy[pos], kv.copy(), np.zeros_like(kv))
    assert rel(y3, y[pos]) < 1e-5
    full = 3.0 * (8 * sh.S * sh.H ** 2 + 6 * sh.S * sh.H * sh.I + 2 * sh.S ** 2 * sh.H)
    assert abs(ob.sample_flops(sh, pos) / (len(pos) / sh.S * full) - 1) < 0.01
