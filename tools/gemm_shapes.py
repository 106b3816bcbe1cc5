"""Times every GEMM of the 7B block step (S=4K, p=1) as the executor launches them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_bench import bench  # noqa: E402

T, H, I = 4096, 4096, 11008
SHAPES = [  # (M, N, K, a_mn, b_mn, epi, name)
    (T, 3 * H, H, False, False, 0, "fwd qkv"), (T, H, H, False, False, 1, "fwd o"),
    (T, 2 * I, H, False, False, 2, "fwd gate|up"), (T, H, I, False, False, 1, "fwd down"),
    (H, I, T, True, True, 3, "wgrad down"), (T, I, H, False, True, 0, "dgrad down"),
    (2 * I, H, T, True, True, 3, "wgrad gu"), (T, H, 2 * I, False, True, 0, "dgrad gu"),
    (H, H, T, True, True, 3, "wgrad o"), (T, H, H, False, True, 0, "dgrad o"),
    (3 * H, H, T, True, True, 3, "wgrad qkv"), (T, H, 3 * H, False, True, 0, "dgrad qkv"),
]
if __name__ == "__main__":
    for M, N, K, a, b, e, name in SHAPES:
        print(name, end=": ")
        bench(M, N, K, a_mn=a, b_mn=b, epi=e if e in (0, 3) else 0)
