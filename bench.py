"""Benchmark of the B200-native ISP transformer block (fwd + bwd), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7b_s32k] [--impl ours|reference]

Default config: 7b_s32k, the configuration BASELINE.md §3 quotes the target on (it fits one GPU).

N > 1 is launched by the driver with torchrun (one process per GPU). Each rank owns S/N
tokens and 1/N of every weight (ISP: sp = ps = N) and runs the block through the C ABI
(libseqplan_isp.so); peers exchange heaps via CUDA IPC (handles swapped over
torch.distributed), collectives are the library's own peer-memory kernels.

metric  block fwd+bwd tokens/s (S / max-over-ranks step time), BASELINE.json
value   device-resident inputs, CUDA events on the compute stream, L2 flushed between
        timed steps (256 MiB write), max over ranks
e2e     same metric through the public API with pinned-host x/dy copied in and y/dx copied
        out every step
roofline  dominant tensor-core kernel of the config (the attention backward at 32K, the GEMMs
        at 4K), per-launch CUDA events in a profiled pass on the launching stream
block_roofline  max(F / (p * bf16 peak), NVLink bytes / 900 GB/s) over the step time
cpu_baseline  the CPU fp32 oracle (oracle/block_oracle.c, OpenMP, all threads) measured on a
        bounded sample of the config (n of the S tokens' full block work), plus the reference's
        own planner functions (oracle/_ref/seqplan_probe --time), single-threaded
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {  # BASELINE.json "configs" (H, heads, S); b = 1, bf16
    "cpu_ref_h512_s1k": dict(H=512, D=8, S=1024),
    "7b_s4k": dict(H=4096, D=32, S=4096),
    "7b_s32k": dict(H=4096, D=32, S=32768),
    "7b_s2k": dict(H=4096, D=32, S=2048),
    "20b_s128k": dict(H=5120, D=40, S=131072),
}
METRIC = "block fwd+bwd tokens/s at 1/2/4/8 B200 (max over ranks); exposed comm %"
SEED = 0x5EED2401


def mlp_dim(h):
    return ((8 * h + 2) // 3 + 255) // 256 * 256


def block_flops(H, S):
    """F = 3 * (8 S H^2 + 6 S H I + 2 S^2 H) (causal attention halved)."""
    I = mlp_dim(H)
    return 3.0 * (8 * S * H * H + 6 * S * H * I + 2 * S * S * H)


def block_nvl_bytes(H, S, p):
    """B_nvl per rank = 3 (p-1)/p e Psi_blk + 8 (p-1)/p e (S/p) H."""
    if p == 1:
        return 0.0
    I = mlp_dim(H)
    psi = 4 * H * H + 3 * H * I + 2 * H
    f = (p - 1) / p
    return 3 * f * 2 * psi + 8 * f * 2 * (S / p) * H


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sust=d.get("bf16_tflops_sustained", 1400.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sust=1400.0, src="fallback")


# ----------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampling (-lms 50) in a background process across the measured region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.06)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        self.samples = [[x.strip() for x in line.split(",")] for line in out.splitlines() if line.strip()]

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = sorted(v for v in (num(s[0]) for s in self.samples) if v is not None)
        mx = max((v for v in (num(s[1]) for s in self.samples) if v is not None), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------------------
# CPU baseline (oracle port, bounded sample — measured, never extrapolated)
# ----------------------------------------------------------------------------------------
class CpuSample:
    """The CPU fp32 oracle's full block fwd + bwd restricted to n token rows spread evenly over the
    S-token sequence (oracle/block_oracle.c ob_block_sample): per-row norms, every GEMM and its
    gradients, RoPE and each row's causal attention against its whole prefix, forward and backward.
    That is n/S of the block's FLOPs (ratio reported), so tokens/s = n / measured seconds is the
    oracle's own throughput on this config. The prefix K|V (the other rows' projections) is
    prepared outside the timed region, like the GPU arm's inputs."""

    def __init__(self, cfg):
        import numpy as np
        from oracle import block as ob
        self.np, self.ob = np, ob
        self.sh = ob.Shape(H=cfg["H"], D=cfg["D"], S=cfg["S"])
        rng = np.random.default_rng(SEED)
        self.rng = rng
        self.w = []
        for shp in self.sh.weight_shapes():
            w = rng.standard_normal(shp, dtype=np.float32) * np.float32(0.02)
            if len(shp) == 1:
                w += 1
            self.w.append(w)
        S, H = self.sh.S, self.sh.H
        self.kv = rng.random((S, 2 * H), dtype=np.float32)
        self.kv -= 0.5
        self.dkv = np.zeros_like(self.kv)
        self.cores = os.cpu_count() or 1
        ob.lib().ob_set_threads(self.cores)

    def positions(self, n):
        S = self.sh.S
        return (self.np.arange(n, dtype=self.np.int64) * (S // n) + (S // n) // 2)

    def run(self, n):
        np = self.np
        pos = self.positions(n)
        x = self.rng.standard_normal((n, self.sh.H), dtype=np.float32)
        dy = self.rng.standard_normal((n, self.sh.H), dtype=np.float32)
        t0 = time.perf_counter()
        self.ob.block_sample(self.sh, self.w, pos, x, dy, self.kv, self.dkv)
        return time.perf_counter() - t0

    def calibrate(self, target_s):
        self.run(8)  # first touch of the weights / K|V pages and the thread pool, untimed
        n = 32
        while True:
            dt = self.run(n)
            if dt >= target_s / 2 or 2 * n > self.sh.S // 8:
                break
            n *= 2
        return n, dt

    def flops_ratio(self, n):
        pos = self.positions(n)
        H, S = self.sh.H, self.sh.S
        return self.ob.sample_flops(self.sh, pos) / (n / S * block_flops(H, S))

    def describe(self, n, dts):
        return (f"oracle fwd+bwd of n={n} of the S={self.sh.S} tokens (every {self.sh.S // n}th position), full "
                f"H={self.sh.H}/{self.sh.D}-head/I={self.sh.I} block work for those rows incl. causal attention "
                f"against their whole prefix ({self.flops_ratio(n):.5f} x n/S of the block FLOPs), "
                f"{len(dts)} runs of {min(dts):.2f}-{max(dts):.2f} s, {self.cores} threads; measured, not extrapolated")


def cpu_baseline(cfg, budget_s=20.0):
    """One bounded measurement of the CPU oracle on this config (bench line's cpu_baseline)."""
    cs = CpuSample(cfg)
    n, _ = cs.calibrate(budget_s / 4)
    dts = [cs.run(n) for _ in range(2)]
    dt = sorted(dts)[len(dts) // 2]
    return {"value": n / dt, "unit": "tokens/s", "cores": cs.cores, "kind": "port",
            "sample": cs.describe(n, dts), "reference_cpu_path": reference_cpu_path(cfg)}


def reference_cpu_path(cfg_name_or_cfg):
    """The reference's own executable code on this path — its planner's estimate_step,
    simulate_forward/backward and run_mempool, compiled from the reference headers into
    oracle/_ref/seqplan_probe — timed single-threaded on this host (µs per call)."""
    name = cfg_name_or_cfg if isinstance(cfg_name_or_cfg, str) else next(
        (k for k, v in CONFIGS.items() if v == cfg_name_or_cfg), None)
    exe = ROOT / "oracle" / "_ref" / "seqplan_probe"
    if name is None or not exe.exists():
        return {"error": "oracle/_ref/seqplan_probe not built"}
    try:
        r = subprocess.run([str(exe), "--time", name], capture_output=True, text=True, timeout=120)
        return json.loads(r.stdout)
    except Exception as ex:  # never sinks the bench line
        return {"error": str(ex)[:200]}


# ----------------------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="7b_s32k", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fused-bwd", action="store_true")
    ap.add_argument("--recompute", action="store_true", help="a = 1: activation recomputation (SURVEY.md §8f item 3)")
    return ap.parse_args()


KERNEL_NAMES = {
    "gemm": "tcgen05 GEMM (all linear-layer GEMMs of the step)",
    "attn_bwd": "tcgen05 causal attention backward (stored-dS pair: attn_bwd_split_kernel<0,0,1> key-tile CTAs "
                "write dK/dV and bulk-store every causal dS tile, attn_bwd_dq_kernel forms dQ = dS K from them; no "
                "atomics; algorithmic FLOPs 4*S^2*Hl, the recomputed S/dP products not counted)",
    "attn_fwd": "tcgen05 causal attention forward (attn_fwd_fa4_kernel; FLOPs 2*S^2*Hl)",
}


def dominant_kernel(by):
    """The tensor-core kernel kind with the largest share of the profiled step (GEMMs at S <= 4K,
    the attention backward at S >= 32K) — the roofline line reports that kernel."""
    cands = [k for k in KERNEL_NAMES if k in by and by[k].get("flops", 0) > 0]
    return max(cands, key=lambda k: by[k]["s"]) if cands else "gemm"


def timeline_exposure(events):
    """Exposed communication from a measured Timeline: |(comm ∪ all-to-all) minus compute| / makespan,
    where compute = compute-stream spans other than the all-to-alls (SURVEY.md §8d cross-check)."""
    def union(iv):
        out = []
        for a, b in sorted(iv):
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out
    comp = union([(e["start"], e["end"]) for e in events if e["stream"] == 0 and e["kind"] != "all_to_all"])
    comm = union([(e["start"], e["end"]) for e in events if e["stream"] == 1 or e["kind"] == "all_to_all"])
    exposed = 0.0
    for a, b in comm:  # subtract the compute cover from each comm interval
        cur = a
        for c, d in comp:
            if d <= cur or c >= b:
                continue
            if c > cur:
                exposed += c - cur
            cur = max(cur, d)
            if cur >= b:
                break
        if cur < b:
            exposed += b - cur
    span = max(e["end"] for e in events) - min(e["start"] for e in events) if events else 0.0
    return {"pct": 100.0 * exposed / span if span > 0 else None, "makespan_ms": span * 1e3,
            "events": len(events), "rank": 0}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def run_reference(args):
    """--impl reference: the reference has no executable block (its CPU path is the planner's
    price model, timed in cpu_baseline.reference_cpu_path), so the CPU restatement of the path
    (oracle port, all host threads) is timed on the same config: every step is one bounded
    sample of the workload (CpuSample: n of the S tokens' full block work), sized to ~2 s."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    cs = CpuSample(cfg)
    n, _ = cs.calibrate(2.0)
    for _ in range(max(1, args.warmup)):
        cs.run(n)
    dts = [cs.run(n) for _ in range(max(1, args.steps))]
    v = n * len(dts) / sum(dts)
    cb = {"value": v, "unit": "tokens/s", "cores": cs.cores, "kind": "port", "sample": cs.describe(n, dts),
          "reference_cpu_path": reference_cpu_path(args.config)}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(dts) / len(dts) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: one ISP block fwd+bwd, H={cfg['H']}, heads={cfg['D']}, "
                                   f"I={mlp_dim(cfg['H'])}, S={cfg['S']}, b=1 (CPU oracle port; each step = "
                                   f"{n} of the {cfg['S']} tokens' block work, ms_per_step is that sample's time)",
                       "sample_tokens_per_step": n, "sample_flops_ratio": cs.flops_ratio(n)},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    import faulthandler
    import signal
    faulthandler.register(signal.SIGUSR1, all_threads=True)  # `kill -USR1` dumps where a run hangs
    # watchdog: a run that is still going after 30 min (normal runs take 1-3 min) dumps every
    # thread's stack to stderr and exits non-zero instead of holding the GPU until an outer timeout
    faulthandler.dump_traceback_later(float(os.environ.get("BENCH_WATCHDOG_S", "1800")), exit=True)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2401_09149_b200 import capi
    from paper_2401_09149_b200.dist import bootstrap_peers

    world, rank, local = dist_env()
    if world != args.gpus:
        world = args.gpus if world == 1 else world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL is plumbing only (IPC-handle exchange, barriers, max over ranks); keep its version
        # banner off stdout, where the one JSON line goes
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    H, D, S = cfg["H"], cfg["D"], cfg["S"]
    T = S // world
    flags = capi.FLAG_FUSED_BWD if args.fused_bwd else 0

    def make_ctx(extra_flags=0):
        blk = capi.IspBlock(H, D, S, world=world, rank=rank, device=local, flags=flags | extra_flags,
                            recompute=args.recompute)
        if world > 1:
            bootstrap_peers(blk, world)
        blk.init_weights(SEED)
        return blk

    blk = make_ctx()
    stream = torch.cuda.Stream(device=dev)
    x = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
    dy = torch.empty_like(x)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    with torch.cuda.stream(stream):
        blk.fill_activation(SEED, 0, x, stream)
        blk.fill_activation(SEED, 1, dy, stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        blk.fwd(x, y, stream)
        blk.bwd(dy, dx, stream)

    def sync_all():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, steps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        sync_all()
        for i in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(i & 0xFF)  # evict L2 between timed steps (outside the events)
                evs[i][0].record(stream)
                fn()
                evs[i][1].record(stream)
        sync_all()
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        t = torch.tensor([ms], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        with torch.cuda.stream(stream):
            step()
    l0 = capi.lib().seqplan_isp_launch_count(blk.h)
    with Clocks(local) as clk:
        ms = timed(step, args.steps)
    launches = capi.lib().seqplan_isp_launch_count(blk.h) - l0
    value = S / (ms / 1e3)
    clocks = clk.summary()

    # ---- end to end through the public API with host buffers ----
    # Every step copies its own inputs x, dy from pinned host memory and reads its results y and dx
    # back. The loop is the one a training job runs: inputs and outputs are double-buffered, step
    # i+1's H2D copies run on a copy stream while step i computes, and step i's D2H copies overlap
    # step i+1. Step i+2 reuses step i's buffers only after step i's D2H has read them (copied[b]).
    # The timed region spans the first copy-in to the last copy-out.
    e2e = None
    if not args.no_e2e:
        hx = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
        hdy = torch.empty_like(hx).pin_memory()
        hy = [torch.empty_like(hx).pin_memory() for _ in range(2)]
        hdx = [torch.empty_like(hx).pin_memory() for _ in range(2)]
        hx.copy_(x.cpu())
        hdy.copy_(dy.cpu())
        xb, dyb = [x, torch.empty_like(x)], [dy, torch.empty_like(dy)]
        yb, dxb = [y, torch.empty_like(y)], [dx, torch.empty_like(dx)]
        copy_in, copy_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        x_ready = [torch.cuda.Event() for _ in range(2)]
        dy_ready = [torch.cuda.Event() for _ in range(2)]
        fwd_done = [torch.cuda.Event() for _ in range(2)]
        step_done = [torch.cuda.Event() for _ in range(2)]
        copied = [torch.cuda.Event() for _ in range(2)]
        for ev in step_done + copied:
            ev.record(stream)

        # x lands first (the forward starts on it while dy is still in flight: the backward waits
        # for dy only), and y leaves as soon as the forward has written it (during the backward)
        def issue_in(i):
            b = i % 2
            copy_in.wait_event(step_done[b])  # step i-2 is done reading this input pair
            with torch.cuda.stream(copy_in):
                xb[b].copy_(hx, non_blocking=True)
                x_ready[b].record(copy_in)
                dyb[b].copy_(hdy, non_blocking=True)
                dy_ready[b].record(copy_in)

        def run(i):
            b = i % 2
            stream.wait_event(x_ready[b])
            stream.wait_event(copied[b])  # step i-2's y / dx have been read back
            blk.fwd(xb[b], yb[b], stream)
            fwd_done[b].record(stream)
            copy_out.wait_event(fwd_done[b])
            with torch.cuda.stream(copy_out):
                hy[b].copy_(yb[b], non_blocking=True)
            stream.wait_event(dy_ready[b])
            blk.bwd(dyb[b], dxb[b], stream)
            step_done[b].record(stream)
            copy_out.wait_event(step_done[b])
            with torch.cuda.stream(copy_out):
                hdx[b].copy_(dxb[b], non_blocking=True)
                copied[b].record(copy_out)

        def e2e_loop(n):
            issue_in(0)
            for i in range(n):
                if i + 1 < n:
                    issue_in(i + 1)
                run(i)
            stream.wait_stream(copy_out)

        with torch.cuda.stream(stream):
            e2e_loop(2)
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.fill_(1)
            e0.record(stream)
            copy_in.wait_event(e0)
            e2e_loop(args.steps)
            e1.record(stream)
        sync_all()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
        nb = T * H * 2
        e2e = {"value": S / (ms_e2e / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": 2 * nb,
               "d2h_bytes_per_step": 2 * nb, "ms_per_step": ms_e2e,
               "copies": "per step and rank: x, dy pinned-host -> device; y, dx device -> pinned host",
               "pipelining": "double-buffered inputs and outputs: step i+1's H2D and step i's D2H overlap compute; "
                             "x copied before dy (the forward waits for x only), y read back during the backward",
               "l2": "flushed once before the loop; per-step working set (weights, activations) > L2"}

    # ---- profiled pass: per-kernel CUDA events (not the headline number) ----
    # HBM: the device pool's own accounting (peak reserved / fragmented) and the
    # device-wide high-water mark of this process
    ps = blk.pool_stats()
    free_b, total_b = torch.cuda.mem_get_info(dev)
    memory = {"pool_peak_reserved_bytes": ps["peak_reserved"], "pool_peak_fragmented_bytes": ps["peak_fragmented"],
              "pool_peak_allocated_bytes": ps["peak_allocated"], "device_used_bytes": total_b - free_b,
              "device_total_bytes": total_b}
    blk.close()
    pblk = make_ctx(capi.FLAG_PROFILE)
    with torch.cuda.stream(stream):
        pblk.fill_activation(SEED, 0, x, stream)
        pblk.fill_activation(SEED, 1, dy, stream)
        for _ in range(2):
            pblk.fwd(x, y, stream)
            pblk.bwd(dy, dx, stream)
    torch.cuda.synchronize(dev)
    recs = pblk.kernel_profile(clear=True)
    nprof = 3
    with torch.cuda.stream(stream):
        for _ in range(nprof):
            pblk.fwd(x, y, stream)
            pblk.bwd(dy, dx, stream)
    torch.cuda.synchronize(dev)
    recs = pblk.kernel_profile(clear=True)
    by = {}
    for r in recs:
        k = by.setdefault(r["kind"], {"flops": 0.0, "bytes": 0.0, "s": 0.0, "n": 0})
        k["flops"] += r["flops"]; k["bytes"] += r["bytes"]; k["s"] += r["seconds"]; k["n"] += 1
    prof_total = sum(k["s"] for k in by.values()) / nprof

    # ---- exposed communication (N > 1): same step with collectives replaced by no-ops ----
    exposed = 0.0 if world == 1 else None
    if world > 1:
        pblk.close()
        sblk = make_ctx(capi.FLAG_SKIP_COMM)
        blk = sblk

        def step_skip():
            sblk.fwd(x, y, stream)
            sblk.bwd(dy, dx, stream)

        for _ in range(3):
            with torch.cuda.stream(stream):
                step_skip()
        ms_skip = timed(step_skip, args.steps)
        exposed = max(0.0, (ms - ms_skip) / ms)
        sblk.close()
    else:
        pblk.close()

    # cross-check of the exposure from the measured CUDA-event Timeline of one step on rank 0
    # (SURVEY.md §8d): time the comm stream (or an all-to-all on the compute stream) is busy
    # while no compute span runs, over the makespan. Never allowed to sink the bench line.
    exposed_tl = None
    if world > 1:
        try:
            tblk = make_ctx(capi.FLAG_TIMELINE)
            for _ in range(2):
                with torch.cuda.stream(stream):
                    tblk.fwd(x, y, stream)
                    tblk.bwd(dy, dx, stream)
            torch.cuda.synchronize(dev)
            exposed_tl = timeline_exposure(tblk.timeline())
            tblk.close()
        except Exception as ex:  # noqa: BLE001
            exposed_tl = {"error": str(ex)[:200]}

    peaks = load_peaks()
    dom = dominant_kernel(by)
    g = by.get(dom, {"flops": 0, "s": 1e-30, "n": 0})
    achieved = g["flops"] / g["s"] / 1e12 if g["s"] > 0 else 0.0
    t_comp = block_flops(H, S) / world / (peaks["bf16"] * 1e12)
    t_nvl = block_nvl_bytes(H, S, world) / 900e9  # 900 GB/s per direction
    t_roof = max(t_comp, t_nvl)
    traffic = None
    tf = ROOT / "profiles" / f"{dom}_traffic_{args.config}.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("traffic_bytes_per_launch")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (index-keyed splitmix64 normals; weights N(0,.02), norms 1+N(0,.02))",
            "config": {"workload": f"{args.config}: one ISP block fwd+bwd (RMSNorm-QKV-RoPE-causal MHA-O-RMSNorm-"
                                   f"SwiGLU), H={H}, heads={D}, I={mlp_dim(H)}, S={S}, b=1",
                       "parallelism": f"isp sp=ps={world}", "global_batch_tokens": S, "seq_len": S,
                       "l2": "flushed between timed steps (256 MiB write); working set > L2",
                       "bwd_policy": "fused" if args.fused_bwd else "selective",
                       "recompute": int(args.recompute)},
            "exposed_comm_pct": None if exposed is None else 100.0 * exposed,
            "exposed_comm_timeline": exposed_tl,
            "block_roofline": {"t_roof_ms": t_roof * 1e3, "bound": "tensor" if t_comp >= t_nvl else "nvlink",
                               "frac": (t_roof * 1e3) / ms, "flops": block_flops(H, S),
                               "nvl_bytes_per_rank": block_nvl_bytes(H, S, world), "nvl_gbs": 900.0,
                               "frac_at_measured_770_gbs": max(t_comp, block_nvl_bytes(H, S, world) / 770e9) * 1e3 / ms,
                               "peak_tflops": peaks["bf16"], "peak_src": peaks["src"]},
            "roofline": {"kernel": KERNEL_NAMES[dom], "bound": "tensor",
                         "achieved": achieved, "peak": peaks["bf16"], "unit": "TFLOP/s",
                         "frac": achieved / peaks["bf16"], "traffic": traffic,
                         "peak_note": f"bf16_tflops burst ({peaks['src']}); vs the sustained "
                                      f"{peaks['bf16_sust']} TF/s: {achieved / peaks['bf16_sust']:.2f} (see clocks)",
                         "share_of_step": (g["s"] / nprof) / prof_total if prof_total else None,
                         "launches_per_step": g["n"] / nprof},
            "kernel_breakdown_ms": {k: v["s"] / nprof * 1e3 for k, v in by.items()},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "memory": memory,
            "e2e": e2e,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(cfg)
            except Exception as ex:  # the baseline must never sink the bench line
                line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
