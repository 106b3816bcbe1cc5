"""Kernel-level parity of the sm_100a attention and RMSNorm kernels vs plain PyTorch fp32."""
import math

import pytest
import torch

from paper_2401_09149_b200 import capi

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def torch_attention(q, k, v):  # [S, h, d] fp32, causal
    S, h, d = q.shape
    s = torch.einsum("qhd,khd->hqk", q, k) / math.sqrt(d)
    mask = torch.ones(S, S, dtype=torch.bool, device=q.device).tril()
    s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)  # [h, S]
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqk,khd->qhd", p, v), lse


def ds_workspace(S, heads, device):
    """Workspace for every head's causal dS tiles (the stored-dS backward)."""
    n = capi.lib().seqplan_isp_debug_attention_ds_bytes(S) * heads
    return torch.empty(n, dtype=torch.uint8, device=device)


@pytest.mark.parametrize("mode", ["split", "ds", "fused"])
@pytest.mark.parametrize("S,heads,d", [(256, 2, 64), (512, 3, 128), (1024, 1, 128), (384, 2, 64)])
def test_attention_fwd_bwd(cuda, S, heads, d, mode, monkeypatch):
    # split: the atomic-free two-role backward (no workspace); ds: the stored-dS backward (key-tile
    # kernel storing the causal dS tiles + the dQ kernel; what the block runs); fused: the opt-in
    # fused backward (dQ reduced with fp32 L2 atomics). ds / fused are d = 128 only.
    if mode != "split" and d != 128:
        pytest.skip("the stored-dS and fused tcgen05 backwards are d = 128")
    if mode == "fused":
        monkeypatch.setenv("SEQPLAN_ISP_ATTN_FUSED_BWD", "1")
    ws = ds_workspace(S, heads, cuda) if mode == "ds" else None
    torch.manual_seed(S + d)
    Hl = heads * d
    qkv = torch.randn(S, 3 * Hl, device=cuda).bfloat16()
    o = torch.empty(S, Hl, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(heads, S, device=cuda)
    q, k, v = qkv[:, :Hl], qkv[:, Hl:2 * Hl], qkv[:, 2 * Hl:]
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    capi.check(l.seqplan_isp_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), 3 * Hl, o.data_ptr(), Hl,
                                             lse.data_ptr(), S, heads, d, None, None, None, None, 0, None, None, st))
    qf, kf, vf = (t.float().view(S, heads, d).requires_grad_(True) for t in (q, k, v))
    ref, ref_lse = torch_attention(qf, kf, vf)
    torch.cuda.synchronize()
    assert rel(o.float().view(S, heads, d), ref) < 1e-2
    assert (lse - ref_lse).abs().max().item() < 2e-2
    # backward
    do = torch.randn(S, Hl, device=cuda).bfloat16()
    ref.backward(do.float().view(S, heads, d))
    dqkv = torch.empty(S, 3 * Hl, device=cuda, dtype=torch.bfloat16)
    delta = torch.empty(heads, S, device=cuda)
    dq_acc = torch.empty(heads * S * d, device=cuda)
    capi.check(l.seqplan_isp_debug_attention_ws(q.data_ptr(), k.data_ptr(), v.data_ptr(), 3 * Hl, o.data_ptr(), Hl,
                                                lse.data_ptr(), S, heads, d, do.data_ptr(), dqkv.data_ptr(),
                                                dqkv[:, Hl:].data_ptr(), dqkv[:, 2 * Hl:].data_ptr(), 3 * Hl,
                                                delta.data_ptr(), dq_acc.data_ptr(),
                                                ws.data_ptr() if ws is not None else None,
                                                ws.numel() if ws is not None else 0, st))
    torch.cuda.synchronize()
    for i, g in enumerate((qf.grad, kf.grad, vf.grad)):
        got = dqkv[:, i * Hl:(i + 1) * Hl].float().view(S, heads, d)
        assert rel(got, g) < 1e-2, (i, rel(got, g))


@pytest.mark.parametrize("T,H", [(64, 512), (300, 4096), (128, 5120), (17, 1024)])
def test_rmsnorm_fwd_bwd(cuda, T, H):
    torch.manual_seed(T)
    x = torch.randn(T, H, device=cuda).bfloat16()
    g = (1 + 0.1 * torch.randn(H, device=cuda)).bfloat16()
    y = torch.empty_like(x)
    rstd = torch.empty(T, device=cuda)
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    capi.check(l.seqplan_isp_debug_rmsnorm(x.data_ptr(), g.data_ptr(), y.data_ptr(), rstd.data_ptr(), None, None,
                                           None, None, T, H, 1e-5, st))
    xf = x.float().requires_grad_(True)
    gf = g.float().requires_grad_(True)
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * gf
    torch.cuda.synchronize()
    assert rel(y.float(), ref) < 5e-3
    dn = torch.randn(T, H, device=cuda).bfloat16()
    dres = torch.randn(T, H, device=cuda).bfloat16()
    dx = torch.empty_like(x)
    dg = torch.zeros(H, device=cuda)
    capi.check(l.seqplan_isp_debug_rmsnorm(x.data_ptr(), g.data_ptr(), None, rstd.data_ptr(), dn.data_ptr(),
                                           dres.data_ptr(), dx.data_ptr(), dg.data_ptr(), T, H, 1e-5, st))
    ref.backward(dn.float())
    torch.cuda.synchronize()
    assert rel(dx.float() - dres.float(), xf.grad) < 1e-2
    assert rel(dg, gf.grad) < 5e-3


def chunked_reference(q, k, v, do, chunk=2048):
    """fp32 causal attention fwd + bwd, query chunk by query chunk (no S x S matrix): o, lse, dq, dk, dv.
    q, k, v, do: [S, d] fp32 of one head."""
    S, d = q.shape
    scale = 1.0 / math.sqrt(d)
    o = torch.empty_like(q); lse = torch.empty(S, device=q.device)
    dq = torch.empty_like(q); dk = torch.zeros_like(k); dv = torch.zeros_like(v)
    for a in range(0, S, chunk):
        b = min(S, a + chunk)
        s = (q[a:b] @ k[:b].t()) * scale
        mask = torch.arange(b, device=q.device)[None, :] > torch.arange(a, b, device=q.device)[:, None]
        s.masked_fill_(mask, float("-inf"))
        l = torch.logsumexp(s, dim=-1)
        p = torch.exp(s - l[:, None])
        o[a:b] = p @ v[:b]
        lse[a:b] = l
        delta = (do[a:b] * o[a:b]).sum(-1)
        dp = do[a:b] @ v[:b].t()
        ds = p * (dp - delta[:, None]) * scale
        dq[a:b] = ds @ k[:b]
        dk[:b] += ds.t() @ q[a:b]
        dv[:b] += p.t() @ do[a:b]
    return o, lse, dq, dk, dv


@pytest.mark.parametrize("S,heads,check_heads", [
    (16384, 8, (0, 5)),    # L2-sized head groups: lpt_grid puts 4 heads in a group, gridDim.z = 2
    (32768, 2, (0, 1)),    # the 7B-32K sequence length
    (131072, 1, (0,)),     # the 20B-128K sequence length: S/128 = 1024 tiles per head
])
@pytest.mark.parametrize("bwd", ["split", "ds"])
def test_attention_long_sequence(cuda, S, heads, check_heads, bwd):
    """The production tcgen05 attention (d = 128) at the BASELINE sequence lengths against a chunked
    fp32 reference: rel-L2 <= 1e-2 on o, dq, dk, dv for the checked heads, |lse| abs error small.
    At S = 128K the backward accumulates dK/dV over 1024 query tiles (SURVEY hard part vi).
    bwd: the two-role kernel, or the stored-dS pair (at 128K one head's dS tiles are 17 GB)."""
    torch.manual_seed(S + heads)
    d = 128
    Hl = heads * d
    qkv = (torch.randn(S, 3 * Hl, device=cuda) * 0.5).bfloat16()
    o = torch.empty(S, Hl, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(heads, S, device=cuda)
    do = torch.randn(S, Hl, device=cuda).bfloat16()
    dqkv = torch.empty(S, 3 * Hl, device=cuda, dtype=torch.bfloat16)
    delta = torch.empty(heads, S, device=cuda)
    dq_acc = torch.empty(heads * S * d, device=cuda)
    q, k, v = qkv[:, :Hl], qkv[:, Hl:2 * Hl], qkv[:, 2 * Hl:]
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    capi.check(l.seqplan_isp_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), 3 * Hl, o.data_ptr(), Hl,
                                             lse.data_ptr(), S, heads, d, None, None, None, None, 0, None, None, st))
    ws = ds_workspace(S, heads, cuda) if bwd == "ds" else None
    capi.check(l.seqplan_isp_debug_attention_ws(q.data_ptr(), k.data_ptr(), v.data_ptr(), 3 * Hl, o.data_ptr(), Hl,
                                                lse.data_ptr(), S, heads, d, do.data_ptr(), dqkv.data_ptr(),
                                                dqkv[:, Hl:].data_ptr(), dqkv[:, 2 * Hl:].data_ptr(), 3 * Hl,
                                                delta.data_ptr(), dq_acc.data_ptr(),
                                                ws.data_ptr() if ws is not None else None,
                                                ws.numel() if ws is not None else 0, st))
    torch.cuda.synchronize()
    del ws
    for h in check_heads:
        cs = slice(h * d, (h + 1) * d)
        qf, kf, vf, dof = (t[:, cs].float() for t in (q, k, v, do))
        ro, rl, rdq, rdk, rdv = chunked_reference(qf, kf, vf, dof)
        assert rel(o[:, cs].float(), ro) < 1e-2, (h, "o")
        assert (lse[h] - rl).abs().max().item() < 2e-2, (h, "lse")
        for i, ref in enumerate((rdq, rdk, rdv)):
            got = dqkv[:, i * Hl:(i + 1) * Hl][:, cs].float()
            e = rel(got, ref)
            assert e < 1e-2, (h, "dq dk dv"[i * 3:i * 3 + 2], e)
        torch.cuda.empty_cache()


@pytest.mark.parametrize("S,heads,group", [(2048, 5, 2), (1024, 4, 3), (4096, 3, 1)])
def test_attention_bwd_ds_head_groups(cuda, S, heads, group):
    """The stored-dS backward with a workspace for `group` heads runs ceil(heads/group) launch pairs
    (head offsets h0); its dq/dk/dv equal the two-role kernel's bit for bit (same fp32 products and
    summation order) and match the fp32 reference."""
    torch.manual_seed(S + heads)
    d = 128
    Hl = heads * d
    qkv = torch.randn(S, 3 * Hl, device=cuda).bfloat16()
    o = torch.empty(S, Hl, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(heads, S, device=cuda)
    do = torch.randn(S, Hl, device=cuda).bfloat16()
    delta = torch.empty(heads, S, device=cuda)
    dq_acc = torch.empty(heads * S * d, device=cuda)
    q, k, v = qkv[:, :Hl], qkv[:, Hl:2 * Hl], qkv[:, 2 * Hl:]
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    capi.check(l.seqplan_isp_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), 3 * Hl, o.data_ptr(), Hl,
                                             lse.data_ptr(), S, heads, d, None, None, None, None, 0, None, None, st))
    ws = torch.full((l.seqplan_isp_debug_attention_ds_bytes(S) * group + 4096,), 0x7f, dtype=torch.uint8,
                    device=cuda)
    outs = []
    for w in (None, ws):
        dqkv = torch.full((S, 3 * Hl), float("nan"), device=cuda, dtype=torch.bfloat16)
        capi.check(l.seqplan_isp_debug_attention_ws(q.data_ptr(), k.data_ptr(), v.data_ptr(), 3 * Hl, o.data_ptr(),
                                                    Hl, lse.data_ptr(), S, heads, d, do.data_ptr(), dqkv.data_ptr(),
                                                    dqkv[:, Hl:].data_ptr(), dqkv[:, 2 * Hl:].data_ptr(), 3 * Hl,
                                                    delta.data_ptr(), dq_acc.data_ptr(),
                                                    w.data_ptr() if w is not None else None,
                                                    w.numel() if w is not None else 0, st))
        outs.append(dqkv)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    qf, kf, vf = (t.float().view(S, heads, d).requires_grad_(True) for t in (q, k, v))
    ref, _ = torch_attention(qf, kf, vf)
    ref.backward(do.float().view(S, heads, d))
    for i, g in enumerate((qf.grad, kf.grad, vf.grad)):
        got = outs[1][:, i * Hl:(i + 1) * Hl].float().view(S, heads, d)
        assert rel(got, g) < 1e-2, (i, rel(got, g))
