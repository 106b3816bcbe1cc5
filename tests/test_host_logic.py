"""CPU tests of host-side logic: device-pool placement vs the reference pool model, and the
multi-process peer bootstrap over a world-size-2 gloo group."""
import os
import subprocess
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def test_device_pool_matches_run_mempool(tmp_path):
    exe = tmp_path / "test_device_pool"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT/'include'}", "-I/usr/local/cuda/include",
                    str(ROOT / "tests" / "cpp" / "test_device_pool.cpp"), "-o", str(exe),
                    "-L/usr/local/cuda/lib64", "-lcudart"], check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True,
                       env={**os.environ, "LD_LIBRARY_PATH": "/usr/local/cuda/lib64"})
    assert r.returncode == 0, r.stdout + r.stderr


class _FakeBlock:
    def __init__(self, rank):
        self.rank = rank
        self.opened = None

    def ipc_handle(self):
        return bytes([self.rank]) * 64

    def open_peers(self, handles):
        self.opened = handles


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2401_09149_b200.dist import bootstrap_peers
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blk = _FakeBlock(rank)
    bootstrap_peers(blk, world)
    q.put((rank, [h[0] for h in blk.opened], [len(h) for h in blk.opened]))
    dist.destroy_process_group()


def test_peer_bootstrap_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, 29611, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, [0, 1], [64, 64]), (1, [0, 1], [64, 64])]


class _FakeNvlsBlock(_FakeBlock):
    """Records the NVLS bootstrap calls; `fail_attach` ranks report an attach failure."""
    def __init__(self, rank, supported=True, fail_attach=()):
        super().__init__(rank)
        self.device = rank
        self.supported, self.fail_attach = supported, fail_attach
        self.calls = []

    def nvls_export(self):
        self.calls.append("export")
        return (4242, 7) if self.supported else None

    def nvls_attach(self, pid, fd):
        self.calls.append(("attach", pid, fd))
        return self.rank not in self.fail_attach

    def nvls_bind(self):
        self.calls.append("bind")
        return True

    def nvls_release(self):
        self.calls.append("release")


def _nvls_worker(rank, world, port, q, supported, fail_attach):
    import torch.distributed as dist
    from paper_2401_09149_b200.dist import bootstrap_peers
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blk = _FakeNvlsBlock(rank, supported, fail_attach)
    bootstrap_peers(blk, world)
    q.put((rank, blk.calls))
    dist.destroy_process_group()


@pytest.mark.parametrize("supported,fail_attach,port", [(True, (), 29612), (False, (), 29613), (True, (1,), 29614)])
def test_nvls_bootstrap_agreement_gloo_world2(supported, fail_attach, port):
    """dist.bootstrap_nvls: rank 0 exports and publishes (pid, fd); the others attach with it (rank
    0 with (0, -1)); binding happens only when every rank attached, and a failure anywhere
    releases NVLS on every rank; an unsupported export stops everyone before attaching."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nvls_worker, args=(r, 2, port, q, supported, fail_attach)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    if not supported:
        assert res == {0: ["export"], 1: []}
    elif not fail_attach:
        assert res == {0: ["export", ("attach", 0, -1), "bind"], 1: [("attach", 4242, 7), "bind"]}
    else:
        assert res == {0: ["export", ("attach", 0, -1), "release"], 1: [("attach", 4242, 7), "release"]}


def test_bench_dominant_kernel_and_timeline_exposure():
    """bench.py's roofline line reports the tensor-core kernel with the largest share of the step,
    and the timeline cross-check counts comm (or all-to-all) time not covered by compute."""
    import bench
    by = {"gemm": {"s": 26.3, "flops": 1.0}, "attn_bwd": {"s": 30.3, "flops": 1.0}, "all_gather": {"s": 50.0, "flops": 0}}
    assert bench.dominant_kernel(by) == "attn_bwd"
    assert bench.dominant_kernel({"gemm": {"s": 3.3, "flops": 1.0}, "attn_bwd": {"s": 0.5, "flops": 1.0}}) == "gemm"
    assert bench.dominant_kernel({}) == "gemm"
    ev = [dict(stream=0, kind="forward", start=0.0, end=1.0), dict(stream=1, kind="all_gather", start=0.5, end=1.5),
          dict(stream=0, kind="all_to_all", start=1.5, end=2.0), dict(stream=0, kind="forward", start=2.0, end=3.0)]
    r = bench.timeline_exposure(ev)
    assert abs(r["pct"] - 100.0 / 3.0) < 1e-9 and r["events"] == 4
