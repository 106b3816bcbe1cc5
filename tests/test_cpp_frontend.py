"""The C++ front-end (include/seqplan/isp_block.hpp) builds against the C-ABI library on CPU,
and on a B200 drives a block whose measured timeline feeds the reference's compare_to_analytic."""
import json
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2401_09149_b200"


def build_demo(out):
    from paper_2401_09149_b200 import capi
    capi.lib()  # ensure the library exists
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT/'include'}", "-I/usr/local/cuda/include",
           str(ROOT / "examples" / "isp_block_demo.cpp"), "-o", str(out), f"-L{LIBDIR}", "-lseqplan_isp",
           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_frontend_compiles_and_links(tmp_path):
    build_demo(tmp_path / "demo")
    assert (tmp_path / "demo").exists()


@pytest.mark.gpu
def test_cpp_frontend_runs_and_feeds_compare_to_analytic(tmp_path, cuda):
    build_demo(tmp_path / "demo")
    r = subprocess.run([str(tmp_path / "demo")], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "LD_LIBRARY_PATH": f"{LIBDIR}:/usr/local/cuda/lib64"})
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["events"] > 0 and d["makespan_ms"] > 0 and d["compute_ms"] > 0
    assert d["pool_reserved"] >= d["pool_allocated"] > 0
