"""Multi-layer stack throughput: per-layer fwd+bwd tokens/s of an L-layer
ISP stack (inter-layer prefetch on one comm stream) against the single block, same harness as
bench.py (CUDA events, L2 flushed between steps, max over ranks). Launch with torchrun for N > 1:
  python -m torch.distributed.run --nproc-per-node 4 tools/stack_bench.py 7b_s4k 4"""
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
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "7b_s4k"
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    cfg = CONFIGS[cfg_name]
    world, rank = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    H, D, S = cfg["H"], cfg["D"], cfg["S"]
    T = S // world
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(device=dev)
    out = {"config": cfg_name, "n_gpus": world, "layers": L}
    for nl in (1, L):
        st = capi.IspStack(nl, H, D, S, world=world, rank=rank, device=local)
        for l in range(nl):
            blk = st.layer(l)
            bootstrap_peers(blk, world)
            blk.init_weights(SEED + l)
        x = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
        st.layer(0).fill_activation(SEED, 0, x)
        dy = torch.empty_like(x)
        st.layer(0).fill_activation(SEED, 1, dy)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for _ in range(3):
                st.fwd(x, y, stream)
                st.bwd(dy, dx, stream)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        with torch.cuda.stream(stream):
            for i in range(steps):
                flush.fill_(i & 0xFF)
                evs[i][0].record(stream)
                st.fwd(x, y, stream)
                st.bwd(dy, dx, stream)
                evs[i][1].record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / steps], device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        out[f"L{nl}_ms_per_step"] = ms.item()
        out[f"L{nl}_tokens_per_s_per_layer"] = S * nl / (ms.item() / 1e3)
        ps = st.layer(0).pool_stats()  # the stack's one device pool (layer 0's)
        out[f"L{nl}_pool_peak_reserved_gib"] = ps["peak_reserved"] / 2**30
        st.close()
        if world > 1:
            dist.barrier()
    out["per_layer_speedup_vs_single_block"] = out[f"L{L}_tokens_per_s_per_layer"] / out["L1_tokens_per_s_per_layer"]
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
