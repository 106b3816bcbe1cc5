"""Prints rank 0's CUDA-event timeline of one block fwd+bwd (SEQPLAN_ISP_FLAG_TIMELINE) and the
reference's compare_to_analytic-style summary. Launch with torchrun for N > 1."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import CONFIGS, SEED  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402
from paper_2401_09149_b200.dist import bootstrap_peers  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7b_s32k"]
    world, rank = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    H, D, S = cfg["H"], cfg["D"], cfg["S"]
    T = S // world
    blk = capi.IspBlock(H, D, S, world=world, rank=rank, device=local, flags=capi.FLAG_TIMELINE)
    bootstrap_peers(blk, world)
    blk.init_weights(SEED)
    x = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
    blk.fill_activation(SEED, 0, x)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        blk.fwd(x, y)
        blk.bwd(x, dx)
    torch.cuda.synchronize()
    if rank == int(os.environ.get("TIMELINE_RANK", 0)):
        ev = blk.timeline()
        comp = [e for e in ev if e["stream"] == 0]
        comm = [e for e in ev if e["stream"] == 1]
        span = max(e["end"] for e in ev) - min(e["start"] for e in ev)
        for e in sorted(ev, key=lambda e: e["start"]):
            print(f"{'C' if e['stream'] == 0 else ' ' * 40 + 'M'} {e['kind']:>15} L{e['layer']} "
                  f"{e['start'] * 1e3:8.3f} -> {e['end'] * 1e3:8.3f} ms")
        print(json.dumps({"makespan_ms": span * 1e3, "compute_busy_ms": sum(e["end"] - e["start"] for e in comp) * 1e3,
                          "comm_busy_ms": sum(e["end"] - e["start"] for e in comm) * 1e3}))
    blk.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
