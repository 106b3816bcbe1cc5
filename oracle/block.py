"""ctypes front-end of oracle/block_oracle.c (CPU fp32 block oracle). TEST INFRASTRUCTURE ONLY.

Parity status: activations/gradients are "parity unpinned" by the reference, which
computes no tensors; this restatement is cross-checked against an
independent PyTorch-autograd restatement in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libblock_oracle.so"
_lib = None

SEED = 0x5EED2401
TID_X, TID_DY, TID_G1, TID_WQKV, TID_WO, TID_G2, TID_WGATE, TID_WUP, TID_WDOWN = range(9)
# weight order = include/seqplan_isp.h SEQPLAN_W_* ; tensor ids per SURVEY.md §8(d)
WEIGHT_TIDS = [TID_G1, TID_WQKV, TID_WO, TID_G2, TID_WGATE, TID_WUP, TID_WDOWN]


class ObShape(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int64), ("D", ctypes.c_int64), ("S", ctypes.c_int64),
                ("I", ctypes.c_int64), ("rope_base", ctypes.c_double), ("eps", ctypes.c_double)]


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(HERE), "oracle"], check=True, capture_output=True)
        l = ctypes.CDLL(str(LIB))
        fp = ctypes.POINTER(ctypes.c_float)
        l.ob_fill.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                              ctypes.c_double, ctypes.c_double, fp]
        l.ob_keyed_normal.restype = ctypes.c_double
        l.ob_keyed_normal.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64]
        l.ob_rope_table.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, fp, fp]
        pp = ctypes.POINTER(fp)
        l.ob_block_isp.argtypes = [ctypes.POINTER(ObShape), ctypes.c_int, pp, fp, fp, fp, fp, pp]
        l.ob_block_sample.argtypes = [ctypes.POINTER(ObShape), pp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                      fp, fp, fp, fp, fp, fp, pp]
        l.ob_set_threads.argtypes = [ctypes.c_int]
        l.ob_max_threads.restype = ctypes.c_int
        _lib = l
    return _lib


def mlp_intermediate_dim(h: int) -> int:
    return ((8 * h + 2) // 3 + 255) // 256 * 256


@dataclass
class Shape:
    H: int
    D: int
    S: int
    I: int = 0
    rope_base: float = 10000.0
    eps: float = 1e-5

    def __post_init__(self):
        if not self.I:
            self.I = mlp_intermediate_dim(self.H)

    def c(self):
        return ObShape(self.H, self.D, self.S, self.I, self.rope_base, self.eps)

    def weight_shapes(self):
        H, I = self.H, self.I
        return [(H,), (3 * H, H), (H, H), (H,), (I, H), (I, H), (H, I)]


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def fill(tid: int, n: int, offset: int = 0, mean: float = 0.0, std: float = 1.0, seed: int = SEED):
    out = np.empty(n, dtype=np.float32)
    lib().ob_fill(seed, tid, offset, n, mean, std, _fp(out))
    return out


def make_weights(shape: Shape, seed: int = SEED):
    """Full fp32 weights: linear N(0, 0.02), norms 1 + N(0, 0.02)."""
    ws = []
    for tid, shp in zip(WEIGHT_TIDS, shape.weight_shapes()):
        n = int(np.prod(shp))
        mean = 1.0 if tid in (TID_G1, TID_G2) else 0.0
        ws.append(fill(tid, n, mean=mean, std=0.02, seed=seed).reshape(shp))
    return ws


def make_activation(shape: Shape, tid: int, seed: int = SEED):
    return fill(tid, shape.S * shape.H, seed=seed).reshape(shape.S, shape.H)


def block(shape: Shape, weights, x, dy, p: int = 1, threads: int = 0):
    """Block fwd+bwd on p simulated ISP ranks. Returns (y, dx, grads[7]) fp32."""
    l = lib()
    if threads:
        l.ob_set_threads(threads)
    ws = [np.ascontiguousarray(w, dtype=np.float32).reshape(-1) for w in weights]
    grads = [np.zeros_like(w) for w in ws]
    x = np.ascontiguousarray(x, dtype=np.float32)
    dy = np.ascontiguousarray(dy, dtype=np.float32)
    y = np.empty_like(x)
    dx = np.empty_like(x)
    FP = ctypes.POINTER(ctypes.c_float)
    warr = (FP * 7)(*[_fp(w) for w in ws])
    garr = (FP * 7)(*[_fp(g) for g in grads])
    sh = shape.c()
    rc = l.ob_block_isp(ctypes.byref(sh), p, warr, _fp(x), _fp(dy), _fp(y), _fp(dx), garr)
    if rc != 0:
        raise ValueError(f"oracle rejected shape {shape} p={p}")
    return y, dx, [g.reshape(s) for g, s in zip(grads, shape.weight_shapes())]


def block_sample(shape: Shape, weights, pos, x_rows, dy_rows, kv, dkv, grads=None):
    """The full fwd + bwd work of the token rows at positions `pos` (bench.py's bounded CPU sample;
    block_oracle.c ob_block_sample). kv [S, 2H]: rotated K|V of every position (the sampled rows'
    own are written in); dkv [S, 2H] accumulates their dK|dV contributions. Returns (y, dx, grads)."""
    l = lib()
    ws = [np.ascontiguousarray(w, dtype=np.float32).reshape(-1) for w in weights]
    if grads is None:
        grads = [np.zeros_like(w) for w in ws]
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    x_rows = np.ascontiguousarray(x_rows, dtype=np.float32)
    dy_rows = np.ascontiguousarray(dy_rows, dtype=np.float32)
    assert kv.dtype == np.float32 and kv.flags.c_contiguous and kv.shape == (shape.S, 2 * shape.H)
    assert dkv.dtype == np.float32 and dkv.flags.c_contiguous and dkv.shape == kv.shape
    y = np.empty_like(x_rows)
    dx = np.empty_like(x_rows)
    FP = ctypes.POINTER(ctypes.c_float)
    warr = (FP * 7)(*[_fp(w) for w in ws])
    garr = (FP * 7)(*[_fp(g) for g in grads])
    sh = shape.c()
    rc = l.ob_block_sample(ctypes.byref(sh), warr, pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pos.size,
                           _fp(x_rows), _fp(dy_rows), _fp(kv), _fp(dkv), _fp(y), _fp(dx), garr)
    if rc != 0:
        raise ValueError(f"oracle rejected sample of {shape}")
    return y, dx, grads


def sample_flops(shape: Shape, pos):
    """Algorithmic FLOPs of block_sample (same convention as the block: 3x the forward, causal
    attention 4*d per head per (query, key<=query) pair in the forward)."""
    H, I = shape.H, shape.I
    per_row = 8 * H * H + 6 * H * I
    attn = 4 * H * float(np.sum(np.asarray(pos, np.float64) + 1))
    return 3.0 * (len(pos) * per_row + attn)


def rope_table(S: int, d: int, base: float = 10000.0):
    c = np.empty((S, d // 2), np.float32)
    s = np.empty((S, d // 2), np.float32)
    lib().ob_rope_table(S, d, base, _fp(c), _fp(s))
    return c, s


def adamw(w, g, m, v, step: int, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
          weight_decay: float = 0.0):
    """One AdamW update of an fp32 shard (torch.optim.AdamW rule: decoupled weight decay, then
    bias-corrected first/second moments). The optimizer step after the path;
    the reference prices it only, as T_update = optimizer-state bytes / 1 TB/s (cost.hpp:292-294).
    Returns (w, m, v) as new float32 arrays; computed in float64."""
    w = np.asarray(w, np.float64); g = np.asarray(g, np.float64)
    m = np.asarray(m, np.float64); v = np.asarray(v, np.float64)
    w = w - lr * weight_decay * w
    m = beta1 * m + (1 - beta1) * g
    v = beta2 * v + (1 - beta2) * g * g
    mh = m / (1 - beta1 ** step)
    vh = v / (1 - beta2 ** step)
    w = w - lr * mh / (np.sqrt(vh) + eps)
    return w.astype(np.float32), m.astype(np.float32), v.astype(np.float32)
