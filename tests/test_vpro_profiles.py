"""Measured VPro curves: every committed
profiles/**/vpro_*.csv loads with the reference's own parser (load_bandwidth_csv_file,
bandwidth.hpp:214-253, compiled from include/seqplan), reproduces its measured points, and
interpolates in log-log space between sizes (bandwidth.hpp:166-196)."""
import json
import math
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CSVS = sorted((ROOT / "profiles").rglob("vpro_*.csv"))


@pytest.fixture(scope="module")
def tool(tmp_path_factory):
    out = tmp_path_factory.mktemp("vpro") / "vpro_lookup"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "vpro_lookup.cpp"),
                    "-o", str(out)], check=True, capture_output=True, text=True)
    return out


@pytest.mark.parametrize("csv", CSVS, ids=[c.name for c in CSVS])
def test_measured_vpro_loads_and_interpolates(tool, csv):
    rows = json.loads(subprocess.run([str(tool), str(csv)], check=True, capture_output=True, text=True).stdout)
    assert rows
    by = {}
    for r in rows:
        assert r["bw"] > 0 and math.isclose(r["lookup"], r["bw"], rel_tol=1e-9)
        assert math.isclose(r["tau"], r["v"] / r["bw"], rel_tol=1e-7)  # %.9g print
        by.setdefault((r["op"], r["p"]), []).append(r)
    for pts in by.values():
        pts.sort(key=lambda r: r["v"])
        for a, b in zip(pts, pts[1:]):
            if b["v"] == 2 * a["v"] or b["v"] > 2 * a["v"]:  # 2v lies inside [a, b]: between the two
                lo, hi = min(a["bw"], b["bw"]), max(a["bw"], b["bw"])
                assert lo * (1 - 1e-9) <= a["lookup_2v"] <= hi * (1 + 1e-9)
        assert math.isclose(pts[-1]["lookup_2v"], pts[-1]["bw"], rel_tol=1e-9)  # clamped past the last size
