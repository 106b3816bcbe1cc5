"""B200-native ISP (hybrid-sharded) transformer block — arXiv 2401.09149 (InternEvo).

The product is ``libseqplan_isp.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/seqplan_isp.h``) plus the C++ ``seqplan::`` headers in ``include/seqplan``.
This Python package is plumbing only: it locates/builds the shared library and
exposes it through ctypes for the tests and ``bench.py``. There is no CPU or
PyTorch fallback — if the library is missing, ``lib()`` raises.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

from .capi import IspBlock, IspGroup, lib, ShapeC, StrategyC, PolicyC, StepStatsC, EventC  # noqa: F401

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libseqplan_isp.so"
