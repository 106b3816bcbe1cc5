"""Bit-exact parity of the ISP collectives' index layout and reduction order (SURVEY.md §8c:
"bit-exact requirements: shard/index layout, A2A permutation").

The Ulysses all-to-all kernels are pure permutations of bf16 rows (
cost.hpp:179-183), so without RoPE they must equal the index permutation exactly
(torch.equal). The gradient reduce-scatter sums the p partials in fixed rank order in fp32 and
then applies the cast / scale (cost.hpp:184-188): it must equal the same fp32 sum done in that
order (torch.equal). Each rank's call is checked on p device buffers standing in for the peers.
"""
import ctypes
import math

import pytest
import torch

from paper_2401_09149_b200 import capi

pytestmark = pytest.mark.gpu


def ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def rope_tables(S, d, dev):
    t = torch.arange(S, dtype=torch.float64, device=dev)[:, None]
    inv = 10000.0 ** (-2.0 * torch.arange(d // 2, dtype=torch.float64, device=dev) / d)
    ang = t * inv[None, :]
    return torch.cos(ang).float().contiguous(), torch.sin(ang).float().contiguous()


@pytest.mark.parametrize("p,H,d,T", [(2, 1024, 128, 96), (4, 1024, 128, 64), (8, 1024, 128, 32), (4, 512, 64, 40),
                                     (8, 4096, 128, 16)])
def test_all_to_all_is_the_index_permutation(cuda, p, H, d, T):
    torch.manual_seed(p * 1000 + H + T)
    parts, S, Hl = 3, p * T, H // p
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    tok = [torch.randn(T, parts * H, device=cuda).bfloat16() for _ in range(p)]
    full = torch.cat(tok).view(S, parts, H)
    heads = []
    for r in range(p):
        dst = torch.empty(S, parts * Hl, device=cuda, dtype=torch.bfloat16)
        capi.check(l.seqplan_isp_debug_all_to_all(p, r, T, H, parts, d, +1, ptrs(tok), dst.data_ptr(), None, None,
                                                  0, st))
        torch.cuda.synchronize()
        want = full[:, :, r * Hl:(r + 1) * Hl].reshape(S, parts * Hl)
        assert torch.equal(dst, want), r
        heads.append(dst)
    # and back: head-sharded on every rank -> token-sharded on this rank is the inverse permutation
    for r in range(p):
        back = torch.empty(T, parts * H, device=cuda, dtype=torch.bfloat16)
        capi.check(l.seqplan_isp_debug_all_to_all(p, r, T, H, parts, d, -1, ptrs(heads), back.data_ptr(), None,
                                                  None, 0, st))
        torch.cuda.synchronize()
        assert torch.equal(back, tok[r]), r


@pytest.mark.parametrize("p", [2, 8])
def test_all_to_all_with_rope_matches_rotation(cuda, p):
    """RoPE applied on the way (q, k parts): the rotation of the permuted rows, within one bf16 rounding."""
    H, d, T, parts = 1024, 128, 64, 3
    S, Hl = p * T, H // p
    torch.manual_seed(7 + p)
    cos, sin = rope_tables(S, d, cuda)
    tok = [torch.randn(T, parts * H, device=cuda).bfloat16() for _ in range(p)]
    full = torch.cat(tok).view(S, parts, H // d, d).float()
    half = d // 2
    a, b = full[..., :half], full[..., half:]
    c, s = cos[:, None, None, :], sin[:, None, None, :]
    rot = torch.cat([a * c - b * s, b * c + a * s], dim=-1)
    want_all = torch.where(torch.arange(parts, device=cuda)[None, :, None, None] < 2, rot, full)
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    for r in range(p):
        dst = torch.empty(S, parts * Hl, device=cuda, dtype=torch.bfloat16)
        capi.check(l.seqplan_isp_debug_all_to_all(p, r, T, H, parts, d, +1, ptrs(tok), dst.data_ptr(),
                                                  cos.data_ptr(), sin.data_ptr(), 2, st))
        torch.cuda.synchronize()
        want = want_all.reshape(S, parts, H)[:, :, r * Hl:(r + 1) * Hl].reshape(S, parts * Hl)
        # one bf16 ulp of the result, plus fp32 rounding of x*c - y*s relative to its operands
        # (the kernel may contract it into an FMA; matters only under cancellation)
        err = (dst.float() - want).abs()
        tol = want.abs() * 2.0 ** -7 + 2.0 ** -20 * full.view(S, parts, H).abs().amax() 
        assert bool((err <= tol).all()), float((err - tol).max())
        # the v part (not rotated) is still an exact permutation
        assert torch.equal(dst.view(S, parts, Hl)[:, 2], full.view(S, parts, H)[:, 2, r * Hl:(r + 1) * Hl].bfloat16())


@pytest.mark.parametrize("f32", [False, True])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_reduce_scatter_is_the_fixed_rank_order_fp32_sum(cuda, p, f32):
    torch.manual_seed(p + 10 * f32)
    shard = 4096 * 3 + 8
    dt = torch.float32 if f32 else torch.bfloat16
    part = [torch.randn(p * shard, device=cuda).to(dt) for _ in range(p)]
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    scale = 0.37
    for r in range(p):
        prior = torch.randn(shard, device=cuda)
        for acc in (0, 1):
            out = prior.clone()
            capi.check(l.seqplan_isp_debug_reduce_scatter(p, r, shard, ptrs(part), int(f32), scale, acc,
                                                          out.data_ptr(), st))
            torch.cuda.synchronize()
            s = torch.zeros(shard, device=cuda)
            for q in range(p):
                s = s + part[q][r * shard:(r + 1) * shard].float()
            want = s * scale
            if acc:
                want = want + prior
            assert torch.equal(out, want), (r, acc)
