"""Independent PyTorch-autograd restatement of the ISP block (fp32, CPU or GPU).

Test infrastructure: cross-checks oracle/block_oracle.c (tests/test_oracle.py) and is the
"plain PyTorch fp32 reference" for kernel-level tests. Same block definition as the oracle
(SURVEY.md Q1): RMSNorm -> QKV -> RoPE(rotate-half) -> causal MHA -> O -> +res -> RMSNorm
-> SwiGLU(gate, up) -> down -> +res.
"""
import math

import torch


def rope_cos_sin(S, d, base=10000.0, device="cpu"):
    t = torch.arange(S, dtype=torch.float64, device=device)[:, None]
    inv = base ** (-2.0 * torch.arange(d // 2, dtype=torch.float64, device=device) / d)
    ang = t * inv[None, :]
    return torch.cos(ang).float(), torch.sin(ang).float()


def rope(x, cos, sin):  # x [S, heads, d]
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([a * c - b * s, b * c + a * s], dim=-1)


def rmsnorm(x, g, eps):
    r = torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps)
    return x * r * g


def block_forward(x, W, D, eps=1e-5, base=10000.0):
    g1, wqkv, wo, g2, wg, wu, wd = W
    S, H = x.shape
    d = H // D
    n1 = rmsnorm(x, g1, eps)
    qkv = n1 @ wqkv.t()
    q, k, v = qkv.split(H, dim=-1)
    cos, sin = rope_cos_sin(S, d, base, x.device)
    q = rope(q.view(S, D, d), cos, sin)
    k = rope(k.view(S, D, d), cos, sin)
    v = v.view(S, D, d)
    s = torch.einsum("qhd,khd->hqk", q, k) / math.sqrt(d)
    mask = torch.ones(S, S, dtype=torch.bool, device=x.device).tril()
    s = s.masked_fill(~mask, float("-inf"))
    p = torch.softmax(s, dim=-1)
    o = torch.einsum("hqk,khd->qhd", p, v).reshape(S, H)
    h = x + o @ wo.t()
    n2 = rmsnorm(h, g2, eps)
    a = torch.nn.functional.silu(n2 @ wg.t()) * (n2 @ wu.t())
    return h + a @ wd.t()


def block_fwd_bwd(x, dy, W, D, eps=1e-5, base=10000.0):
    x = x.clone().requires_grad_(True)
    Wt = [w.clone().requires_grad_(True) for w in W]
    y = block_forward(x, Wt, D, eps, base)
    y.backward(dy)
    return y.detach(), x.grad.detach(), [w.grad.detach() for w in Wt]
