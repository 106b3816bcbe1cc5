"""Push all-gather rounds through the real context (development): per-GPU incoming GB/s of the
forward weight set (and both sets). Launch with torchrun, e.g. 4 ranks:
  python -m torch.distributed.run --nproc-per-node 4 tools/gather_bench.py 7b_s4k"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import CONFIGS, SEED, mlp_dim  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402
from paper_2401_09149_b200.dist import bootstrap_peers  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7b_s4k"]
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    H, D, S = cfg["H"], cfg["D"], cfg["S"]
    blk = capi.IspBlock(H, D, S, world=world, rank=rank, device=local)
    bootstrap_peers(blk, world)
    blk.init_weights(SEED)
    l = capi.lib()
    l.seqplan_isp_debug_gather_bench.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                 ctypes.POINTER(ctypes.c_float)]
    I = mlp_dim(H)
    psi = 4 * H * H + 3 * H * I + 2 * H
    for both in (0, 1):
        ms = ctypes.c_float()
        capi.check(l.seqplan_isp_debug_gather_bench(blk.h, 10, both, ctypes.byref(ms)), blk.h, "gather_bench")
        t = torch.tensor([ms.value], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        incoming = (1 + both) * psi * 2 * (world - 1) / world
        if rank == 0:
            print(f"p={world} sets={1 + both}: {t.item():.3f} ms/round, {incoming / t.item() / 1e6:.0f} GB/s incoming "
                  f"per GPU (ag kind={os.environ.get('SEQPLAN_ISP_AG_KIND', 'default')} ctas={os.environ.get('SEQPLAN_ISP_AG_CTAS', 'default')})", flush=True)
    blk.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
