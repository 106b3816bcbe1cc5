"""Quick GEMM timing (CUDA events) for development; not part of the bench contract."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_09149_b200 import capi

def bench(M, N, K, a_mn=False, b_mn=False, epi=0, iters=20):
    dev = torch.device("cuda")
    A = torch.randn(K, M, device=dev).bfloat16() if a_mn else torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if b_mn else torch.randn(N, K, device=dev).bfloat16()
    out = torch.empty(M, N, device=dev, dtype=torch.float32 if epi == 3 else torch.bfloat16)
    for _ in range(3):
        capi.debug_gemm(A, B, out, M, N, K, a_mn=a_mn, b_mn=b_mn, epi=epi)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        capi.debug_gemm(A, B, out, M, N, K, a_mn=a_mn, b_mn=b_mn, epi=epi)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    tf = 2 * M * N * K / ms / 1e9
    # torch reference
    At = A.t() if a_mn else A
    Bt = B if b_mn else B.t()
    for _ in range(3): torch.matmul(At, Bt)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): torch.matmul(At, Bt)
    e.record(); torch.cuda.synchronize()
    ms2 = s.elapsed_time(e) / iters
    print(f"M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} epi={epi}: {ms:.3f} ms {tf:.0f} TF/s | torch {ms2:.3f} ms {2*M*N*K/ms2/1e9:.0f} TF/s", flush=True)

if __name__ == "__main__":
    for (M, N, K) in [(4096, 12288, 4096), (4096, 4096, 4096), (4096, 22016, 4096), (4096, 4096, 11008), (8192, 8192, 8192)]:
        bench(M, N, K)
    bench(4096, 4096, 12288, b_mn=True)
    bench(12288, 4096, 4096, a_mn=True, b_mn=True, epi=3)
