"""Development sweep: tile-order group (SEQPLAN_GEMM_GROUP_M) per GEMM shape of the 7B block,
CUDA events with an L2 flush before each timed launch (not the bench contract)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_09149_b200 import capi  # noqa: E402


def run(M, N, K, gm, iters=5, mn=False):
    os.environ["SEQPLAN_GEMM_GROUP_M"] = str(gm)
    # mn: the weight-gradient form, A stored [K, M] and B stored [K, N] (MN-major)
    a = torch.randn(K, M, device="cuda").bfloat16() if mn else torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16() if mn else torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    capi.debug_gemm(a, b, out, M, N, K, a_mn=mn, b_mn=mn)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(iters):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        capi.debug_gemm(a, b, out, M, N, K, a_mn=mn, b_mn=mn)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    ms = tot / iters
    return ms, 2.0 * M * N * K / ms / 1e9


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "wgrad":
        for M, N, K in [(4096, 11008, 32768), (12288, 4096, 32768), (22016, 4096, 32768), (4096, 4096, 32768),
                        (4096, 11008, 4096), (12288, 4096, 4096)]:
            res = []
            for gm in (2, 4, 8, 16, 32):
                ms, tf = run(M, N, K, gm, mn=True)
                res.append(f"gm{gm}: {ms:.3f} ms {tf:.0f}")
            print(f"wgrad M={M} N={N} K={K}: " + " | ".join(res), flush=True)
        sys.exit(0)
    shapes = [(4096, 4096, 11008), (4096, 4096, 22016), (4096, 12288, 4096), (4096, 4096, 4096), (4096, 22016, 4096),
              (32768, 4096, 11008), (32768, 4096, 22016), (32768, 12288, 4096)]
    for M, N, K in shapes:
        res = []
        for gm in (2, 4, 8, 16, 32):
            ms, tf = run(M, N, K, gm)
            res.append(f"gm{gm}: {ms:.3f} ms {tf:.0f}")
        print(f"M={M} N={N} K={K}: " + " | ".join(res), flush=True)
