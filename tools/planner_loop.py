"""Measured B200 profiles -> the reference planner.

Run under torchrun (N >= 2) or alone. Rank 0 writes
  profiles/vpro_<config>_p<N>.csv   — all-gather / reduce-scatter / all-to-all effective bandwidth
                                      in the reference's CSV schema (bandwidth.hpp:214-253), message
                                      sizes in the reference's tau convention (cost.hpp:177-188)
  profiles/planner_<config>_p<N>.json — estimate_step (via tools/planner_check) vs measurement
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import CONFIGS, SEED, mlp_dim  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402
from paper_2401_09149_b200.dist import bootstrap_peers  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "7b_s4k"
    cfg = CONFIGS[name]
    world, rank = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    H, D, S = cfg["H"], cfg["D"], cfg["S"]
    T = S // world
    blk = capi.IspBlock(H, D, S, world=world, rank=rank, device=local, flags=capi.FLAG_PROFILE | capi.FLAG_TIMELINE)
    bootstrap_peers(blk, world)
    blk.init_weights(SEED)
    x = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
    blk.fill_activation(SEED, 0, x)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(2):
        blk.fwd(x, y)
        blk.bwd(x, dx)
    torch.cuda.synchronize()
    blk.kernel_profile(clear=True)
    n = 5
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(n):
        blk.fwd(x, y)
        blk.bwd(x, dx)
    s1.record()
    torch.cuda.synchronize()
    step = s0.elapsed_time(s1) / n / 1e3
    recs = blk.kernel_profile(clear=True)
    tl = blk.timeline()
    fwd_compute = sum(e["end"] - e["start"] for e in tl if e["stream"] == 0 and e["kind"] == "forward")
    agg = {}
    for r in recs:
        a = agg.setdefault(r["kind"], [0.0, 0.0])
        a[0] += r["seconds"] / n
        a[1] += r["bytes"] / n
    if rank == 0:
        prof_dir = Path(os.environ.get("PLANNER_OUT", str(ROOT / "profiles")))
        prof_dir.mkdir(exist_ok=True)
        e = 2
        I = mlp_dim(H)
        psi_ref = 12 * H * H + 2 * H
        act = e * S * H
        rows = []
        if world > 1:
            # tau convention: message = full layer parameter / activation bytes (cost.hpp:177-188)
            t_ag = agg.get("all_gather", [0, 0])[0] / 2  # two gathers (fwd, bwd) per step
            t_rs = agg.get("reduce_scatter", [0, 0])[0]
            if t_ag > 0:
                rows.append(("all-gather", world, "intra", e * psi_ref, e * psi_ref / t_ag))
            if t_rs > 0:
                rows.append(("reduce-scatter", world, "intra", e * psi_ref, e * psi_ref / t_rs))
            t_a2a = agg.get("all_to_all", [0, 0])[0]
            if t_a2a > 0:  # pull all-to-all path: 4 per step, total 8 act-equivalents
                rows.append(("all-to-all", world, "intra", act, 8 * act / t_a2a))
            else:  # fused into the producers' epilogues: priced at the measured NVLink peer rate
                rows.append(("all-to-all", world, "intra", act, 770e9))
        csv = prof_dir / f"vpro_{name}_p{world}.csv"
        with open(csv, "w") as f:
            f.write("# measured on B200 by tools/planner_loop.py (CUDA events, contended with compute)\n")
            f.write("op,participants,axis,message_bytes,bandwidth_bytes_per_sec\n")
            # one NVSwitch box: every peer is equally close, but place_groups classifies the ps
            # group of the single-box ISP plan as inter -> same curve on both axes
            for r in rows:
                for axis in ("intra", "inter"):
                    f.write(f"{r[0]},{r[1]},{axis},{int(r[3])},{r[4]:.6e}\n")
            if not rows:
                f.write("all-gather,2,intra,1,9.0e11\n")
        exe = ROOT / "tools" / "_planner_check"
        subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT/'include'}", str(ROOT / "tools" / "planner_check.cpp"),
                        "-o", str(exe)], check=True)
        out = subprocess.run([str(exe), str(csv), str(H), str(D), str(S), str(world), f"{fwd_compute:.9g}",
                              f"{step:.9g}"], capture_output=True, text=True, check=True).stdout
        res = json.loads(out)
        res.update({"config": name, "measured_fwd_compute_s": fwd_compute,
                    "kernel_s_per_step": {k: v[0] for k, v in agg.items()}})
        (prof_dir / f"planner_{name}_p{world}.json").write_text(json.dumps(res, indent=1))
        print(json.dumps(res))
    blk.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
