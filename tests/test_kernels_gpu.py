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


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("S,heads,d", [(256, 2, 64), (512, 3, 128), (1024, 1, 128), (384, 2, 64)])
def test_attention_fwd_bwd(cuda, S, heads, d, split, monkeypatch):
    # split: the opt-in two-kernel backward (dK/dV kernel + CTA-pair dQ kernel), d = 128 only
    if split and d != 128:
        pytest.skip("split backward is d = 128")
    if split:
        monkeypatch.setenv("SEQPLAN_ISP_ATTN_SPLIT_BWD", "1")
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
    capi.check(l.seqplan_isp_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), 3 * Hl, o.data_ptr(), Hl,
                                             lse.data_ptr(), S, heads, d, do.data_ptr(), dqkv.data_ptr(),
                                             dqkv[:, Hl:].data_ptr(), dqkv[:, 2 * Hl:].data_ptr(), 3 * Hl,
                                             delta.data_ptr(), dq_acc.data_ptr(), st))
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
