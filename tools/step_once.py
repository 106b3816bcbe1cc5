"""Runs (warm-up + 1) block steps of a config on cuda:0 — a short command for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS, SEED  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402

if __name__ == "__main__":
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7b_s4k"]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    H, D, S = cfg["H"], cfg["D"], cfg["S"]
    blk = capi.IspBlock(H, D, S, world=1)
    blk.init_weights(SEED)
    x = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)
    blk.fill_activation(SEED, 0, x)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(steps):
        blk.fwd(x, y)
        blk.bwd(x, dx)
    torch.cuda.synchronize()
    print("ok")
