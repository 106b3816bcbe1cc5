"""The C-ABI library loads without a GPU and exports every symbol include/seqplan_isp.h declares."""
import ctypes
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "seqplan_isp.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(seqplan_isp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_block_api():
    names = declared()
    for must in ("seqplan_isp_ctx_create", "seqplan_isp_block_fwd", "seqplan_isp_block_bwd",
                 "seqplan_isp_pool_stats", "seqplan_isp_timeline", "seqplan_isp_open_peers"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2401_09149_b200 import capi
    lib = capi.lib()  # builds with nvcc if needed; loading needs no GPU
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2401_09149_b200" / "libseqplan_isp.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (seqplan_isp_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert isinstance(getattr(lib, n), ctypes._CFuncPtr)


def test_sm100a_cubin_has_tcgen05_and_tma():
    """The GEMM is a real tcgen05/TMA kernel (SASS UTCHMMA / UTMALDG / LDTM)."""
    sass = subprocess.run(["cuobjdump", "-sass", str(ROOT / "paper_2401_09149_b200" / "libseqplan_isp.so")],
                          capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem


def test_invalid_arguments_are_rejected_without_gpu():
    from paper_2401_09149_b200 import capi
    l = capi.lib()
    h = capi.c_vp()
    sh = capi.make_shape(512, 7, 1024)  # 512 % 7 != 0 -> invalid model config
    st = l.seqplan_isp_ctx_create(1, 3, 0, ctypes.byref(sh), None, None, 0, ctypes.byref(h))
    assert st == 1 and not h.value  # rank >= world


def test_unsupported_micro_batching_is_refused_without_gpu():
    """A legal ISP plan the executor does not run (b != 1 sequences per micro-batch, gs / oss groups)
    is refused with SEQPLAN_ISP_ERR_UNSUPPORTED instead of silently running b = 1 (isp_block.cpp
    create_ctx); n > 1 micro-batches are run (gradient accumulation, test_block_gpu.py)."""
    from paper_2401_09149_b200 import capi
    l = capi.lib()
    sh = capi.make_shape(512, 8, 1024)
    for field, val in (("micro_batch", 2), ("micro_batch", 4)):
        st = capi.StrategyC(micro_batch=1, micro_batch_num=1, recompute=0, pp=1, dp=1, tp=1, sp=2, ps=2, gs=1, oss=1)
        setattr(st, field, val)
        h = capi.c_vp()
        rc = l.seqplan_isp_ctx_create(2, 0, 0, ctypes.byref(sh), ctypes.byref(st), None, 0, ctypes.byref(h))
        assert rc == 4 and not h.value, (field, rc)
    # an illegal plan stays "invalid" (sp must equal the world size)
    st = capi.StrategyC(micro_batch=1, micro_batch_num=1, recompute=0, pp=1, dp=1, tp=1, sp=1, ps=2, gs=1, oss=1)
    h = capi.c_vp()
    assert l.seqplan_isp_ctx_create(2, 0, 0, ctypes.byref(sh), ctypes.byref(st), None, 0, ctypes.byref(h)) == 1
