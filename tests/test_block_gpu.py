"""Block-level parity: the sm_100a ISP block (through the C ABI) vs the CPU fp32 oracle.

Bar (BASELINE.json north_star): rel-L2 <= 1e-2 for bf16 activations and gradients.
p = 1 runs one context; p = 2/4 run the single-process group mode (p ranks on one
GPU, lock-step phases, peer buffers = each other's heaps) — the same kernels the
multi-process path runs, with the collectives inline. Weight-gradient shards are
compared per rank against the oracle's reduce-scattered shards (ShardingLayout E/F).
"""
import numpy as np
import pytest
import torch

from oracle import block as ob
from paper_2401_09149_b200 import capi

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


_CACHE = {}


def oracle_case(H, D, S):
    key = (H, D, S)
    if key not in _CACHE:
        sh = ob.Shape(H=H, D=D, S=S)
        w = ob.make_weights(sh)
        # the GPU consumes bf16 activations: feed the oracle the same rounded values
        x = torch.from_numpy(ob.make_activation(sh, ob.TID_X)).bfloat16().float().numpy()
        dy = torch.from_numpy(ob.make_activation(sh, ob.TID_DY)).bfloat16().float().numpy()
        y, dx, g = ob.block(sh, w, x, dy, p=1)
        _CACHE[key] = (sh, w, x, dy, y, dx, g)
    return _CACHE[key]


def load_weights(blk, w, p, r):
    for t in range(7):
        flat = w[t].reshape(-1)
        per = flat.size // p
        blk.set_weight_shard(t, flat[r * per:(r + 1) * per])


def check_grads(blocks, g, p):
    for t in range(7):
        flat = g[t].reshape(-1)
        per = flat.size // p
        got = np.concatenate([b.grad_shard(t) for b in blocks])
        assert got.size == flat.size
        e = rel(got, flat)
        assert e <= TOL, (capi.W_NAMES[t], e)


@pytest.mark.parametrize("H,D,S", [(512, 8, 1024), (1024, 8, 512)])
def test_block_p1(cuda, H, D, S):
    sh, w, x, dy, y_ref, dx_ref, g_ref = oracle_case(H, D, S)
    blk = capi.IspBlock(H, D, S, world=1)
    load_weights(blk, w, 1, 0)
    xd = torch.from_numpy(x).to(cuda).bfloat16()
    dyd = torch.from_numpy(dy).to(cuda).bfloat16()
    y = torch.empty_like(xd)
    dx = torch.empty_like(xd)
    blk.fwd(xd, y)
    blk.bwd(dyd, dx)
    torch.cuda.synchronize()
    assert rel(y.float().cpu(), y_ref) <= TOL
    assert rel(dx.float().cpu(), dx_ref) <= TOL
    check_grads([blk], g_ref, 1)
    # a second step is identical (buffers recycled by the pool, no stale state)
    y2 = torch.empty_like(xd)
    dx2 = torch.empty_like(xd)
    blk.fwd(xd, y2)
    blk.bwd(dyd, dx2)
    torch.cuda.synchronize()
    assert torch.equal(y2, y) and torch.equal(dx2, dx)
    blk.close()


@pytest.mark.parametrize("fused_a2a", [False, True])
@pytest.mark.parametrize("p,H,D,S", [(2, 512, 8, 1024), (4, 512, 8, 1024), (2, 1024, 8, 1024), (4, 1024, 8, 1024),
                                     (8, 1024, 8, 2048)])  # p = 8: the north-star degree, on one GPU
def test_block_group(cuda, p, H, D, S, fused_a2a, monkeypatch):
    if fused_a2a and H // D != 128:
        pytest.skip("the fused all-to-all is for head dim 128")
    if fused_a2a:  # the all-to-all fused into the producers' epilogues
        monkeypatch.setenv("SEQPLAN_ISP_FUSED_A2A", "1")
    sh, w, x, dy, y_ref, dx_ref, g_ref = oracle_case(H, D, S)
    grp = capi.IspGroup(H, D, S, world=p)
    blocks = [grp.rank(r) for r in range(p)]
    for r, b in enumerate(blocks):
        load_weights(b, w, p, r)
    T = S // p
    xs = [torch.from_numpy(x[r * T:(r + 1) * T]).to(cuda).bfloat16() for r in range(p)]
    dys = [torch.from_numpy(dy[r * T:(r + 1) * T]).to(cuda).bfloat16() for r in range(p)]
    ys = [torch.empty_like(t) for t in xs]
    dxs = [torch.empty_like(t) for t in xs]
    grp.fwd(xs, ys)
    grp.bwd(dys, dxs)
    torch.cuda.synchronize()
    assert rel(torch.cat(ys).float().cpu(), y_ref) <= TOL
    assert rel(torch.cat(dxs).float().cpu(), dx_ref) <= TOL
    check_grads(blocks, g_ref, p)
    grp.close()


def test_device_init_matches_oracle_generator(cuda):
    H, D, S, p = 512, 8, 1024, 2
    grp = capi.IspGroup(H, D, S, world=p)
    sh = ob.Shape(H=H, D=D, S=S)
    full = ob.make_weights(sh, seed=1234)
    for r in range(p):
        b = grp.rank(r)
        b.init_weights(1234)
        for t in range(7):
            flat = full[t].reshape(-1)
            per = flat.size // p
            got = b.weight_shard(t)
            np.testing.assert_allclose(got, flat[r * per:(r + 1) * per], rtol=0, atol=1e-6)
    grp.close()


def test_pool_trace_replays_through_run_mempool_model(cuda):
    """The device pool places buffers with the reference's best-fit pool: the bytes it
    actually reserved for the general pool equal run_mempool's replay of its own trace."""
    H, D, S = 512, 8, 1024
    blk = capi.IspBlock(H, D, S, world=1, policy=capi.make_policy(pinned=False, premap=False))
    blk.init_weights(7)
    x = torch.randn(S, H, device=cuda).bfloat16()
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        blk.fwd(x, y)
        blk.bwd(x, dx)
    torch.cuda.synchronize()
    st = blk.pool_stats()
    assert st["peak_reserved"] >= st["reserved"] > 0
    assert st["reserved"] == st["allocated"] + st["free_cached"] + st["fragmented"]
    # the reference's run_mempool (mempool.hpp:285-387) replaying the pool's own recorded
    # alloc/free trace reserves exactly the bytes the device pool reserved
    rep = blk.pool_replay()
    assert rep["peak_reserved"] == st["peak_reserved"], (rep, st)
    blk.close()


def test_adamw_step_matches_oracle(cuda):
    """Optimizer step after the path: two AdamW steps on every fp32 master
    shard with the device gradient shards match the oracle's AdamW, and the next forward uses
    the refreshed bf16 working shards."""
    H, D, S = 512, 8, 1024
    sh, w, x, dy, y_ref, dx_ref, g_ref = oracle_case(H, D, S)
    blk = capi.IspBlock(H, D, S, world=1)
    load_weights(blk, w, 1, 0)
    xd = torch.from_numpy(x).bfloat16().to(cuda)
    dyd = torch.from_numpy(dy).bfloat16().to(cuda)
    y, dx = torch.empty_like(xd), torch.empty_like(xd)
    blk.fwd(xd, y)
    blk.bwd(dyd, dx)
    torch.cuda.synchronize()
    y0 = y.float().cpu().numpy().copy()
    w0 = [blk.weight_shard(t) for t in range(7)]
    g = [blk.grad_shard(t) for t in range(7)]
    lr, wd = 1e-3, 0.1
    blk.adamw_step(lr, 1, weight_decay=wd)
    blk.adamw_step(lr, 2, weight_decay=wd)
    torch.cuda.synchronize()
    for t in range(7):
        m = np.zeros_like(g[t]); v = np.zeros_like(g[t])
        ref, m, v = ob.adamw(w0[t], g[t], m, v, 1, lr, weight_decay=wd)
        ref, m, v = ob.adamw(ref, g[t], m, v, 2, lr, weight_decay=wd)
        got = blk.weight_shard(t)
        assert np.abs(got - ref).max() <= 1e-6 + 1e-5 * np.abs(ref).max(), capi.W_NAMES[t]
        assert np.abs(got - w0[t]).max() > 0  # the step moved every tensor
    blk.fwd(xd, y)
    torch.cuda.synchronize()
    assert rel(y.float().cpu().numpy(), y0) > 1e-4  # the refreshed working shards are used
    blk.close()


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def stack_oracle(sh, ws, x, dy):
    """L-layer chain of the oracle block with the GPU's bf16 rounding at layer boundaries."""
    ys, xs = [], [x]
    for w in ws:
        y, _, _ = ob.block(sh, w, xs[-1], np.zeros_like(xs[-1]), p=1)
        ys.append(y)
        xs.append(_bf16(y))
    g_in, grads = dy, [None] * len(ws)
    for l in reversed(range(len(ws))):
        _, dx, g = ob.block(sh, ws[l], xs[l], g_in, p=1)
        grads[l] = g
        g_in = _bf16(dx)
    return ys[-1], dx, grads


@pytest.mark.parametrize("H,D,S", [(512, 8, 1024), (1024, 8, 512)])
def test_stack_two_layers_p1(cuda, H, D, S):
    """Multi-layer stack: 2 layers with independent weights through
    seqplan_isp_stack_fwd/bwd vs the oracle block chained twice."""
    sh, w0, x, dy, _, _, _ = oracle_case(H, D, S)
    w1 = ob.make_weights(sh, seed=ob.SEED + 1)
    y_ref, dx_ref, g_ref = stack_oracle(sh, [w0, w1], x, dy)
    st = capi.IspStack(2, H, D, S)
    for l, w in enumerate((w0, w1)):
        load_weights(st.layer(l), w, 1, 0)
    xd = torch.from_numpy(x).bfloat16().to(cuda)
    dyd = torch.from_numpy(dy).bfloat16().to(cuda)
    y, dx = torch.empty_like(xd), torch.empty_like(xd)
    for _ in range(2):  # second step: buffers / flags reused
        st.fwd(xd, y)
        st.bwd(dyd, dx)
    torch.cuda.synchronize()
    assert rel(y.float().cpu(), y_ref) <= TOL
    assert rel(dx.float().cpu(), dx_ref) <= TOL
    for l in range(2):
        for t in range(7):
            e = rel(st.layer(l).grad_shard(t), g_ref[l][t].reshape(-1))
            assert e <= TOL, (l, capi.W_NAMES[t], e)
    st.close()


def stack_oracle_n(sh, ws, x, dy):
    """The oracle block chained len(ws) times, with the GPU's bf16 rounding at layer boundaries."""
    def bf16(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()
    xs = [x]
    for w in ws:
        yl, _, _ = ob.block(sh, w, xs[-1], np.zeros_like(xs[-1]), p=1)
        xs.append(bf16(yl))
    g_in, grads = dy, [None] * len(ws)
    for l in reversed(range(len(ws))):
        _, dxl, g = ob.block(sh, ws[l], xs[l], g_in, p=1)
        grads[l] = g
        g_in = bf16(dxl)
    return yl, dxl, grads


@pytest.mark.parametrize("H,D,S", [(512, 8, 1024), (1024, 8, 512)])
def test_block_recompute_p1(cuda, H, D, S):
    """Activation recomputation (a = 1; cost.hpp:139, 227): only the block
    input survives the forward, the backward re-runs the forward on the re-gathered weights.
    Same results as the oracle; far fewer bytes live between the passes than at a = 0."""
    sh, w, x, dy, y_ref, dx_ref, g_ref = oracle_case(H, D, S)
    xd = torch.from_numpy(x).bfloat16().to(cuda)
    dyd = torch.from_numpy(dy).bfloat16().to(cuda)
    live = {}
    for a in (0, 1):
        blk = capi.IspBlock(H, D, S, world=1, recompute=bool(a))
        load_weights(blk, w, 1, 0)
        y, dx = torch.empty_like(xd), torch.empty_like(xd)
        for _ in range(2):
            blk.fwd(xd, y)
            torch.cuda.synchronize()
            live[a] = blk.pool_stats()["allocated"]
            blk.bwd(dyd, dx)
        torch.cuda.synchronize()
        assert rel(y.float().cpu(), y_ref) <= TOL
        assert rel(dx.float().cpu(), dx_ref) <= TOL
        check_grads([blk], g_ref, 1)
        blk.close()
    T = S
    saved = T * H * 2 * 5 + S * 3 * H * 2  # n1, o, h, n2, a|gu (>= 1 of them), qkv heads
    assert live[0] - live[1] >= saved, live


@pytest.mark.parametrize("p", [2, 4])
def test_block_group_recompute(cuda, p):
    """a = 1 in group mode (p ranks on one GPU): the recomputed forward repeats both all-to-alls."""
    H, D, S = 1024, 8, 1024
    sh, w, x, dy, y_ref, dx_ref, g_ref = oracle_case(H, D, S)
    grp = capi.IspGroup(H, D, S, world=p, flags=capi.FLAG_RECOMPUTE)
    blocks = [grp.rank(r) for r in range(p)]
    T = S // p
    for r, b in enumerate(blocks):
        load_weights(b, w, p, r)
    xs = [torch.from_numpy(x[r * T:(r + 1) * T]).bfloat16().to(cuda) for r in range(p)]
    dys = [torch.from_numpy(dy[r * T:(r + 1) * T]).bfloat16().to(cuda) for r in range(p)]
    ys = [torch.empty_like(v) for v in xs]
    dxs = [torch.empty_like(v) for v in xs]
    for _ in range(2):
        grp.fwd(xs, ys)
        grp.bwd(dys, dxs)
    torch.cuda.synchronize()
    assert rel(torch.cat(ys).float().cpu(), y_ref) <= TOL
    assert rel(torch.cat(dxs).float().cpu(), dx_ref) <= TOL
    check_grads(blocks, g_ref, p)
    grp.close()


def test_stack_recompute_consolidated_pool(cuda):
    """4-layer stack at a = 1 with checkpoints packed two to a region (consolidate_every_k_mlp = 2)
    and the gradient arena pre-mapped: parity with the oracle chain, and the device pool
    reserves exactly what the reference's run_mempool reserves over the pool's own trace in the
    first step; afterwards the device recycles its packed regions (flat) while the reference's
    never-returned regions grow."""
    H, D, S, L = 512, 8, 1024, 4
    sh, w0, x, dy, _, _, _ = oracle_case(H, D, S)
    ws = [w0] + [ob.make_weights(sh, seed=ob.SEED + l) for l in range(1, L)]
    y_ref, dx_ref, g_ref = stack_oracle_n(sh, ws, x, dy)
    pol = capi.make_policy(pinned=False, consolidate=2, premap=True)
    st = capi.IspStack(L, H, D, S, policy=pol, recompute=True)
    for l, w in enumerate(ws):
        load_weights(st.layer(l), w, 1, 0)
    xd = torch.from_numpy(x).bfloat16().to(cuda)
    dyd = torch.from_numpy(dy).bfloat16().to(cuda)
    y, dx = torch.empty_like(xd), torch.empty_like(xd)
    st.fwd(xd, y)
    st.bwd(dyd, dx)
    torch.cuda.synchronize()
    dev1, rep1 = st.layer(0).pool_stats(), st.layer(0).pool_replay()
    assert dev1["peak_reserved"] == rep1["peak_reserved"], (dev1, rep1)
    assert dev1["reserved"] == dev1["allocated"] + dev1["free_cached"] + dev1["fragmented"]
    for _ in range(2):
        st.fwd(xd, y)
        st.bwd(dyd, dx)
    torch.cuda.synchronize()
    dev3, rep3 = st.layer(0).pool_stats(), st.layer(0).pool_replay()
    assert dev3["peak_reserved"] == dev1["peak_reserved"]
    assert rep3["peak_reserved"] > dev3["peak_reserved"]
    assert rel(y.float().cpu(), y_ref) <= TOL
    assert rel(dx.float().cpu(), dx_ref) <= TOL
    for l in range(L):
        for t in range(7):
            e = rel(st.layer(l).grad_shard(t), g_ref[l][t].reshape(-1))
            assert e <= TOL, (l, capi.W_NAMES[t], e)
    st.close()


@pytest.mark.parametrize("p", [2, 4])
def test_block_fused_swiglu_bwd_epilogue(cuda, p, monkeypatch):
    """Opt-in SwiGLU backward inside the down-projection dgrad epilogue (SEQPLAN_ISP_FUSE_SWIGLU_BWD=1)
    gives the same block results as the separate kernel path."""
    monkeypatch.setenv("SEQPLAN_ISP_FUSE_SWIGLU_BWD", "1")
    H, D, S = 1024, 8, 1024
    sh, w, x, dy, y_ref, dx_ref, g_ref = oracle_case(H, D, S)
    grp = capi.IspGroup(H, D, S, world=p)
    blocks = [grp.rank(r) for r in range(p)]
    for r, b in enumerate(blocks):
        load_weights(b, w, p, r)
    T = S // p
    xs = [torch.from_numpy(x[r * T:(r + 1) * T]).bfloat16().to(cuda) for r in range(p)]
    dys = [torch.from_numpy(dy[r * T:(r + 1) * T]).bfloat16().to(cuda) for r in range(p)]
    ys = [torch.empty_like(v) for v in xs]
    dxs = [torch.empty_like(v) for v in xs]
    grp.fwd(xs, ys)
    grp.bwd(dys, dxs)
    torch.cuda.synchronize()
    assert rel(torch.cat(dxs).float().cpu(), dx_ref) <= TOL
    check_grads(blocks, g_ref, p)
    grp.close()


@pytest.mark.parametrize("n", [2, 3])
def test_micro_batches_accumulate_gradients(cuda, n):
    """Strategy::micro_batch_num = n (GS accumulation, cost.hpp:202-204): the n fwd/bwd calls of a
    step add their weight gradients into the fp32 shards (the first overwrites), so a step's
    gradients equal the oracle's summed over its micro-batches; the next step starts afresh."""
    H, D, S = 1024, 8, 512
    sh = ob.Shape(H=H, D=D, S=S)
    w = ob.make_weights(sh)
    mbs = []
    for k in range(n):  # independent micro-batches (keyed with seeds derived from the step seed)
        x = torch.from_numpy(ob.make_activation(sh, ob.TID_X, seed=ob.SEED + 17 * k)).bfloat16()
        dy = torch.from_numpy(ob.make_activation(sh, ob.TID_DY, seed=ob.SEED + 17 * k)).bfloat16()
        mbs.append((x, dy))
    g_sum = None
    for x, dy in mbs:
        _, _, g = ob.block(sh, w, x.float().numpy(), dy.float().numpy(), p=1)
        g_sum = [t.reshape(-1).copy() for t in g] if g_sum is None else [a + t.reshape(-1) for a, t in zip(g_sum, g)]
    blk = capi.IspBlock(H, D, S, world=1, micro_batches=n)
    load_weights(blk, w, 1, 0)
    for step in range(2):  # the second step must not keep the first step's gradients
        for x, dy in mbs:
            xd, dyd = x.to(cuda), dy.to(cuda)
            y, dx = torch.empty_like(xd), torch.empty_like(xd)
            blk.fwd(xd, y)
            blk.bwd(dyd, dx)
        torch.cuda.synchronize()
        for t in range(7):
            e = rel(blk.grad_shard(t), g_sum[t])
            assert e <= TOL, (step, capi.W_NAMES[t], e)
    blk.close()
