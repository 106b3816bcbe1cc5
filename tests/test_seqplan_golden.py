"""Bit-exact parity of include/seqplan (layout, schedule, pool) with the reference.

tests/golden/seqplan_golden.json was produced by oracle/seqplan_probe.cpp compiled
against the reference's own headers (/root/reference/proj/include, `make -C oracle
golden`). Here the same probe is compiled against *our* headers and its output must
match byte for byte: shard layouts (strategy.hpp:52-62), plan legality and group
axes (strategy.hpp:72-99, placement.hpp:39-59), comm/compute prices (cost.hpp),
timelines (overlap_sim.hpp) and pool traces (mempool.hpp), doubles printed %.17g.

The drop-in gate additionally compiles the reference's own unit tests against our
headers when /root/reference is mounted (this container only).
"""
import json
import os
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden" / "seqplan_golden.json"
REF_TESTS = Path("/root/reference/proj/tests")
CXX = shutil.which("g++") or "g++"


def _build(src, out, extra=()):
    cmd = [CXX, "-std=c++20", "-O2", f"-I{ROOT/'include'}", *extra, str(src), "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


@pytest.fixture(scope="module")
def probe_output(tmp_path_factory):
    exe = tmp_path_factory.mktemp("probe") / "seqplan_probe"
    _build(ROOT / "oracle" / "seqplan_probe.cpp", exe)
    return subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout


def test_probe_matches_reference_golden_bytes(probe_output):
    assert probe_output.strip() == GOLDEN.read_text().strip()


def test_golden_known_values():
    """Spot values documented in SURVEY.md §8 (a5, a16, a19) and BASELINE.md."""
    g = json.loads(GOLDEN.read_text())
    lay = g["layouts"]["7b_s4k/p8"]
    # QKV, O, gate/up/down, norm per-rank shard sizes at p=8, H=4096 (a5)
    assert [t[2] for t in lay[:7]] == [512, 6291456, 2097152, 512, 5636096, 5636096, 5636096]
    assert lay[7][2] == 25166848 and lay[8] == 11008
    plan = g["plans"]["7b_s32k/p8"]
    assert plan["other_buffers"] == 805339136  # 768 MiB pinned double buffer (a16)
    pools = g["pools"]["7b_s32k_L32_p8"]
    assert [pools[k]["peak_reserved"] for k in ("base", "pinned", "consolidate3", "premap", "all")] == [
        2116042752, 2518712320, 1780498432, 2149597184, 2216722432]
    assert pools["base"]["peak_fragmented"] == 369098752  # 16 x 22 MiB
    assert pools["consolidate3"]["peak_fragmented"] == 0
    p20 = g["pools"]["20b_s128k_L60_p8"]
    assert p20["base"]["peak_reserved"] == 15577665536
    assert p20["base"]["peak_fragmented"] == 3523215360


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference not mounted (GPU box)")
@pytest.mark.parametrize("suite", ["test_mempool", "test_overlap_sim", "test_strategy",
                                   "test_placement", "test_cost", "test_bandwidth"])
def test_reference_unit_tests_against_our_headers(suite, tmp_path):
    """Drop-in gate: the reference's own doctest suites, compiled against include/seqplan."""
    exe = tmp_path / suite
    _build(REF_TESTS / f"{suite}.cpp", exe, extra=[f"-I{ROOT/'tests'/'cpp'}"])
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
