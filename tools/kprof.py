"""Per-launch kernel profile of one block step (CUDA events, SEQPLAN_ISP_FLAG_PROFILE) on rank 0:
kind, algorithmic FLOPs / bytes and achieved TF/s or GB/s per launch. Launch with torchrun for N > 1.
  python -m torch.distributed.run --nproc-per-node 2 tools/kprof.py 7b_s4k"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import CONFIGS, SEED  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402
from paper_2401_09149_b200.dist import bootstrap_peers  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7b_s4k"]
    world, rank = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    H, D, S = cfg["H"], cfg["D"], cfg["S"]
    T = S // world
    blk = capi.IspBlock(H, D, S, world=world, rank=rank, device=local, flags=capi.FLAG_PROFILE | (capi.FLAG_SKIP_COMM if os.environ.get("KPROF_SKIP") == "1" else 0))
    bootstrap_peers(blk, world)
    blk.init_weights(SEED)
    x = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    blk.fill_activation(SEED, 0, x)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        blk.fwd(x, y)
        blk.bwd(x, dx)
    torch.cuda.synchronize()
    blk.kernel_profile(clear=True)
    blk.fwd(x, y)
    blk.bwd(x, dx)
    torch.cuda.synchronize()
    recs = blk.kernel_profile(clear=True)
    if rank == 0:
        tot = sum(r["seconds"] for r in recs)
        for r in recs:
            rate = f"{r['flops'] / r['seconds'] / 1e12:7.1f} TF/s" if r["flops"] else \
                f"{r['bytes'] / r['seconds'] / 1e9:7.1f} GB/s"
            print(f"{r['kind']:>16} {r['seconds'] * 1e3:8.3f} ms  flops {r['flops']:.3e}  bytes {r['bytes']:.3e}  {rate}")
        print(f"total {tot * 1e3:.3f} ms over {len(recs)} profiled launches")
    blk.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
