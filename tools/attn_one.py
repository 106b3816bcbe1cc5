"""Runs one attention fwd+bwd (S, heads from argv) — a short command for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.attn_bench import run  # noqa: E402

if __name__ == "__main__":
    S, h = int(sys.argv[1]), int(sys.argv[2])
    run(S, h, 128, iters=1)
