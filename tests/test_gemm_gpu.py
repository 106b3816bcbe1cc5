"""tcgen05 GEMM parity vs a plain PyTorch fp32 reference of the same op.

Covers the three linear-layer shapes (fwd NT, dgrad with MN-major B, wgrad with
MN-major A and B) and every fused epilogue. bf16 inputs, fp32 accumulation:
tolerance rel-L2 <= 2e-3 against fp32 math on the same bf16 inputs.
"""
import pytest
import torch

from paper_2401_09149_b200 import capi

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = a.float(); b = b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def _rand(*shape, dev):
    return torch.randn(*shape, device=dev).to(torch.bfloat16)


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 128, 192), (512, 768, 512), (384, 1536, 320)])
def test_gemm_layouts(cuda, a_mn, b_mn, M, N, K):
    A = _rand(M, K, dev=cuda)
    B = _rand(N, K, dev=cuda)
    a_store = A.t().contiguous() if a_mn else A
    b_store = B.t().contiguous() if b_mn else B
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    capi.debug_gemm(a_store, b_store, out, M, N, K, a_mn=a_mn, b_mn=b_mn, epi=0)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    assert rel_l2(out, ref) < 4e-3


def test_gemm_resid_and_scale(cuda):
    M, N, K = 256, 512, 256
    A, B, R = _rand(M, K, dev=cuda), _rand(N, K, dev=cuda), _rand(M, N, dev=cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    capi.debug_gemm(A, B, out, M, N, K, epi=1, resid=R, scale=0.5)
    torch.cuda.synchronize()
    ref = 0.5 * (A.float() @ B.float().t()) + R.float()
    assert rel_l2(out, ref) < 4e-3


def test_gemm_swiglu(cuda):
    M, K, I = 256, 256, 384
    A = _rand(M, K, dev=cuda)
    Wg, Wu = _rand(I, K, dev=cuda), _rand(I, K, dev=cuda)
    # interleave 32-row blocks (kGuBlock): gate blk j, up blk j, ...
    Wgu = torch.stack([Wg.view(I // 32, 32, K), Wu.view(I // 32, 32, K)], 1).reshape(2 * I, K)
    gu = torch.empty(M, 2 * I, device=cuda, dtype=torch.bfloat16)
    a = torch.empty(M, I, device=cuda, dtype=torch.bfloat16)
    capi.debug_gemm(A, Wgu, gu, M, 2 * I, K, epi=2, out2=a)
    torch.cuda.synchronize()
    g = A.float() @ Wg.float().t()
    u = A.float() @ Wu.float().t()
    gu_v = gu.view(M, I // 32, 2, 32)
    assert rel_l2(gu_v[:, :, 0].reshape(M, I), g) < 4e-3
    assert rel_l2(gu_v[:, :, 1].reshape(M, I), u) < 4e-3
    assert rel_l2(a, torch.nn.functional.silu(g) * u) < 1e-2


def test_gemm_f32_interleaved_wgrad(cuda):
    # dW_gu = dgu^T x  (A MN-major, B MN-major) de-interleaved into fp32 gate/up grads
    T, I, H = 256, 192, 256
    dgu = _rand(T, 2 * I, dev=cuda)
    x = _rand(T, H, dev=cuda)
    g_out = torch.full((I, H), 1.0, device=cuda)
    u_out = torch.full((I, H), 1.0, device=cuda)
    capi.debug_gemm(dgu, x, g_out, 2 * I, H, T, a_mn=True, b_mn=True, epi=3, out_b=u_out,
                    scale=0.25, accumulate=True, interleave64=True)
    torch.cuda.synchronize()
    full = 0.25 * (dgu.float().t() @ x.float())  # [2I, H] interleaved
    fv = full.view(I // 32, 2, 32, H)
    assert rel_l2(g_out - 1.0, fv[:, 0].reshape(I, H)) < 2e-3
    assert rel_l2(u_out - 1.0, fv[:, 1].reshape(I, H)) < 2e-3


def test_gemm_large(cuda):
    M, N, K = 4096, 12288, 4096
    A, B = _rand(M, K, dev=cuda), _rand(N, K, dev=cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    capi.debug_gemm(A, B, out, M, N, K)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    assert rel_l2(out, ref) < 4e-3


@pytest.mark.parametrize("pbn", ["128", "256"])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_pair_tile_widths(cuda, pbn, a_mn, b_mn, monkeypatch):
    """CTA-pair kernel with 256 x 128 and 256 x 256 tiles, every operand layout and epilogue."""
    monkeypatch.setenv("SEQPLAN_GEMM_PAIR_BN", pbn)
    M, N, K = 768, 1280, 448
    A, B, R = _rand(M, K, dev=cuda), _rand(N, K, dev=cuda), _rand(M, N, dev=cuda)
    a_store = A.t().contiguous() if a_mn else A
    b_store = B.t().contiguous() if b_mn else B
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    capi.debug_gemm(a_store, b_store, out, M, N, K, a_mn=a_mn, b_mn=b_mn, epi=1, resid=R, scale=0.5)
    torch.cuda.synchronize()
    assert rel_l2(out, 0.5 * (A.float() @ B.float().t()) + R.float()) < 4e-3
    o32 = torch.full((M, N), 1.0, device=cuda)
    capi.debug_gemm(a_store, b_store, o32, M, N, K, a_mn=a_mn, b_mn=b_mn, epi=3, scale=0.25, accumulate=True)
    torch.cuda.synchronize()
    assert rel_l2(o32 - 1.0, 0.25 * (A.float() @ B.float().t())) < 2e-3
    I = 640  # gate|up interleaved in 32-row blocks, SwiGLU epilogue
    Wg, Wu = _rand(I, K, dev=cuda), _rand(I, K, dev=cuda)
    Wgu = torch.stack([Wg.view(I // 32, 32, K), Wu.view(I // 32, 32, K)], 1).reshape(2 * I, K)
    gu = torch.empty(M, 2 * I, device=cuda, dtype=torch.bfloat16)
    a = torch.empty(M, I, device=cuda, dtype=torch.bfloat16)
    capi.debug_gemm(A, Wgu, gu, M, 2 * I, K, epi=2, out2=a)
    torch.cuda.synchronize()
    g = A.float() @ Wg.float().t()
    u = A.float() @ Wu.float().t()
    assert rel_l2(a, torch.nn.functional.silu(g) * u) < 1e-2


@pytest.mark.parametrize("M,N,K", [(4096, 4096, 4096), (4096, 12288, 1024), (2048, 14336, 2048)])
@pytest.mark.parametrize("epi", [0, 1, 3])
def test_gemm_split_last_wave(cuda, M, N, K, epi, monkeypatch):
    """Tile counts that leave a partial last wave (256 = 3 x 74 + 34, 768 = 10 x 74 + 28,
    448 = 6 x 74 + 4) take the split-K path: the trailing tiles' K-ranges run concurrently and the
    last finisher adds the others' fp32 partials before the fused epilogue. Also run twice to
    check the self-resetting arrival flags."""
    monkeypatch.setenv("SEQPLAN_GEMM_SPLIT", "1")
    A, B, R = _rand(M, K, dev=cuda), _rand(N, K, dev=cuda), _rand(M, N, dev=cuda)
    ref = A.float() @ B.float().t()
    for _ in range(2):
        if epi == 3:
            out = torch.full((M, N), 1.0, device=cuda)
            capi.debug_gemm(A, B, out, M, N, K, epi=3, scale=0.5, accumulate=True)
            torch.cuda.synchronize()
            assert rel_l2(out - 1.0, 0.5 * ref) < 2e-3
        else:
            out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
            capi.debug_gemm(A, B, out, M, N, K, epi=epi, resid=R if epi == 1 else None)
            torch.cuda.synchronize()
            assert rel_l2(out, ref + (R.float() if epi == 1 else 0)) < 4e-3


@pytest.mark.parametrize("M,I,K", [(256, 384, 256), (512, 1024, 320)])
def test_gemm_swiglu_bwd_epilogue(cuda, M, I, K):
    """Down-projection dgrad with the SwiGLU backward fused into the epilogue (EPI_SWIGLU_BWD):
    da = dy Wd (bf16-rounded, never stored) -> dgu (gate|up interleaved in 32-column blocks) from
    the saved gu; matches the unfused formula on the same bf16 inputs."""
    A, B = _rand(M, K, dev=cuda), _rand(I, K, dev=cuda)
    gu = _rand(M, 2 * I, dev=cuda)
    dgu = torch.empty(M, 2 * I, device=cuda, dtype=torch.bfloat16)
    capi.debug_gemm(A, B, dgu, M, I, K, epi=4, resid=gu)
    torch.cuda.synchronize()
    da = (A.float() @ B.float().t()).bfloat16().float()
    guv = gu.float().view(M, I // 32, 2, 32)
    g, u = guv[:, :, 0].reshape(M, I), guv[:, :, 1].reshape(M, I)
    sg = torch.sigmoid(g)
    dg = da * u * sg * (1 + g * (1 - sg))
    du = da * g * sg
    out = dgu.float().view(M, I // 32, 2, 32)
    assert rel_l2(out[:, :, 0].reshape(M, I), dg) < 1e-2
    assert rel_l2(out[:, :, 1].reshape(M, I), du) < 1e-2
