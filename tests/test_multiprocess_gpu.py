"""Multi-process ISP block over real CUDA-IPC peer mappings (one process per GPU).

Skipped unless >= 2 GPUs are visible. Each rank's y / dx slice and fp32 gradient shard
must match the CPU oracle within rel-L2 1e-2 (selective and fused backward)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_rows(out):
    """Every JSON object the ranks printed; ranks share one stdout, so two rows can end up on one
    line — decode objects one after another instead of line by line."""
    dec, rows, i = json.JSONDecoder(), [], out.find("{")
    while i >= 0:
        try:
            obj, end = dec.raw_decode(out, i)
        except json.JSONDecodeError:  # a brace in a log line
            i = out.find("{", i + 1)
            continue
        if isinstance(obj, dict) and "rank" in obj:
            rows.append(obj)
        i = out.find("{", end)
    return rows


def _run(n, H, D, S, mode="selective", env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + n + (7 if mode == 'fused' else 0) + (20 if H == 1024 else 0) + (40 + 3 * int(env.get('SEQPLAN_ISP_PUSH', '0')) + 5 * int(env.get('SEQPLAN_ISP_FUSED_A2A', '0')) if env else 0)}",
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), str(H), str(D), str(S), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = _json_rows(r.stdout)
    assert len(rows) == n
    return rows


@pytest.mark.parametrize("mode", ["selective", "fused"])
@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("H", [512, 1024])  # head dim 64 (pull all-to-all) and 128 (fused into epilogues)
def test_multiprocess_parity(n, mode, H):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    for row in _run(n, H, 8, 1024, mode):
        for k, v in row.items():
            if k not in ("rank", "timeline_events"):
                assert v <= 1e-2, (row["rank"], k, v)
        assert row["timeline_events"] > 0


@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_parity_fused_a2a(n):
    """The Ulysses all-to-all fused into the producers' epilogues (SEQPLAN_ISP_FUSED_A2A=1)."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    for row in _run(n, 1024, 8, 1024, "selective", env={"SEQPLAN_ISP_FUSED_A2A": "1"}):
        for k, v in row.items():
            if k not in ("rank", "timeline_events"):
                assert v <= 1e-2, (row["rank"], k, v)


@pytest.mark.parametrize("push", ["0", "1"])
def test_multiprocess_parity_forced_transport(push):
    """Both weight-traffic transports at p = 2: copy-engine pull (default at p = 2) and the
    bulk-copy push into the pinned double buffer (default at p >= 4)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    for row in _run(2, 1024, 8, 1024, "selective", env={"SEQPLAN_ISP_PUSH": push}):
        for k, v in row.items():
            if k not in ("rank", "timeline_events"):
                assert v <= 1e-2, (row["rank"], k, v)


@pytest.mark.parametrize("push", ["0", "1"])
@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_stack_parity(n, push):
    """2-layer stack with inter-layer prefetch on one comm stream, both
    weight-traffic transports, vs the oracle block chained twice."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29560 + n + 10 * int(push)}",
           os.path.join(ROOT, "tests", "mp_stack_worker.py"), "1024", "8", "1024", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, "SEQPLAN_ISP_PUSH": push})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = _json_rows(r.stdout)
    assert len(rows) == n
    for row in rows:
        for k, v in row.items():
            if k != "rank":
                assert v <= 1e-2, (row["rank"], k, v)


@pytest.mark.parametrize("push", ["0", "1"])
@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_stack_recompute_parity(n, push):
    """Activation recomputation (a = 1) in a 2-layer stack over real peers:
    each layer's backward re-runs its forward from the checkpoint on the re-gathered weights;
    checkpoints packed two to a region (consolidate_every_k_mlp = 2); both transports."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29580 + n + 10 * int(push)}",
           os.path.join(ROOT, "tests", "mp_stack_worker.py"), "1024", "8", "1024", "2", "recompute"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, "SEQPLAN_ISP_PUSH": push})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = _json_rows(r.stdout)
    assert len(rows) == n
    for row in rows:
        for k, v in row.items():
            if k != "rank":
                assert v <= 1e-2, (row["rank"], k, v)


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("H", [512, 1024])
def test_multiprocess_parity_ce_a2a(n, H):
    """Ulysses all-to-all on the copy engines (SEQPLAN_ISP_A2A_CE=1): one strided 2-D copy per
    source rank, RoPE applied in the QKV GEMM epilogue before the exchange, inverse RoPE after
    the backward exchange; head dim 64 and 128."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    for row in _run(n, H, 8, 1024, "selective", env={"SEQPLAN_ISP_A2A_CE": "1"}):
        for k, v in row.items():
            if k not in ("rank", "timeline_events"):
                assert v <= 1e-2, (row["rank"], k, v)


@pytest.mark.parametrize("mode", ["steps", "steps_adamw"])
@pytest.mark.parametrize("n,push", [(2, "0"), (4, "1")])
def test_multiprocess_back_to_back_steps(n, push, mode):
    """The path bench.py times: no flags, 3 fwd/bwd steps back to back without host sync, with
    and without an AdamW update after steps 1 and 2, copy-engine pull at p = 2 and push at p = 4;
    step 3's outputs and gradients (rel-L2 <= 1e-2) vs the oracle at the weights step 3 used."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29620 + n + 10 * (mode == 'steps_adamw')}",
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), "1024", "8", "1024", mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={**os.environ, "SEQPLAN_ISP_PUSH": push})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = _json_rows(r.stdout)
    assert len(rows) == n
    for row in rows:
        for k, v in row.items():
            if k != "rank":
                assert v <= 1e-2, (row["rank"], k, v)


@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_parity_ag_into_gemm(n):
    """The forward all-gather of Wqkv fused into the QKV GEMM (SEQPLAN_ISP_AG_GEMM=1): the peer
    slices' B operands are TMA-loaded straight from the peers' working shards over NVLink."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29660 + n}",
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), "1024", "8", "1024", "steps"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={**os.environ, "SEQPLAN_ISP_AG_GEMM": "1"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = _json_rows(r.stdout)
    assert len(rows) == n
    for row in rows:
        for k, v in row.items():
            if k != "rank":
                assert v <= 1e-2, (row["rank"], k, v)


def test_multiprocess_parity_8_ranks_on_4_gpus():
    """World size 8 through the multi-process production path (push transport, memop barriers,
    pull all-to-all, 8 peers) with two ranks per GPU — the p = 8 code path on a 4-GPU box. The
    ranks of one GPU time-slice, so this is a correctness check only."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29588",
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), "1024", "8", "1024", "selective"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={**os.environ, "MP_RANKS_PER_GPU": "2"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = _json_rows(r.stdout)
    assert len(rows) == 8
    for row in rows:
        for k, v in row.items():
            if k not in ("rank", "timeline_events"):
                assert v <= 1e-2, (row["rank"], k, v)


def test_multiprocess_nvls_reduce_scatter():
    """The NVLink SHARP reduce-scatter at p = 4 (the default there where the GPUs support
    multicast): every rank reports it active, and the block matches the oracle."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    rows = _run(4, 1024, 8, 1024, "selective", env={"SEQPLAN_ISP_PUSH": "1", "SEQPLAN_ISP_NVLS": "1",
                                                     "MP_REPORT_NVLS": "1"})
    for row in rows:
        assert row.pop("nvls_active") == 1, row
        for k, v in row.items():
            if k not in ("rank", "timeline_events"):
                assert v <= 1e-2, (row["rank"], k, v)
