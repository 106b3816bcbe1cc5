"""ctypes bindings of include/seqplan_isp.h (plumbing for tests and bench.py).

This mirrors what a maintainer would bind from the reference side (see
INTEGRATION.md): plain pointers, sizes and POD structs; torch is used only to
own device memory and streams.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
_LIB_PATH = _PKG / "libseqplan_isp.so"
_lib = None

c_int, c_i64, c_u32, c_u64, c_vp, c_f, c_d = (ctypes.c_int, ctypes.c_int64, ctypes.c_uint32,
                                             ctypes.c_uint64, ctypes.c_void_p, ctypes.c_float,
                                             ctypes.c_double)


class ShapeC(ctypes.Structure):
    _fields_ = [("hidden_dim", c_i64), ("heads", c_i64), ("seq_len", c_i64), ("ffn_dim", c_i64),
                ("rope_base", c_d), ("norm_eps", c_d)]


class StrategyC(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("micro_batch", "micro_batch_num", "recompute", "pp", "dp",
                                     "tp", "sp", "ps", "gs", "oss")]


class PolicyC(ctypes.Structure):
    _fields_ = [("pinned_comm_pool", ctypes.c_int32), ("consolidate_every_k_mlp", c_i64),
                ("grad_premap", ctypes.c_int32), ("capacity", c_i64)]


class AdamWC(ctypes.Structure):
    _fields_ = [("lr", c_d), ("beta1", c_d), ("beta2", c_d), ("eps", c_d), ("weight_decay", c_d), ("step", c_i64)]


class StepStatsC(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("reserved", "allocated", "free_cached", "fragmented",
                                     "peak_reserved", "peak_fragmented", "peak_allocated")]


class EventC(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_int32), ("kind", ctypes.c_int32), ("layer", c_i64),
                ("start_s", c_d), ("end_s", c_d)]


class KernelRecC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("flops", c_d), ("bytes", c_d), ("seconds", c_d)]


K_NAMES = ["gemm", "attn_fwd", "attn_bwd", "all_gather", "reduce_scatter", "all_to_all", "elementwise"]

STATUS = {0: "ok", 1: "invalid argument", 2: "runtime error", 3: "out of memory",
          4: "unsupported"}

W_NORM1, W_QKV, W_O, W_NORM2, W_GATE, W_UP, W_DOWN = range(7)
W_NAMES = ["norm1", "qkv", "o", "norm2", "gate", "up", "down"]
FLAG_NO_OVERLAP, FLAG_FUSED_BWD, FLAG_TIMELINE, FLAG_SKIP_COMM, FLAG_PROFILE = 1, 2, 4, 8, 16
FLAG_RECOMPUTE = 32  # a = 1 where no Strategy is passed (group mode)
ERR_UNSUPPORTED = 4
EV_NAMES = ["forward", "grad_input", "grad_weight", "all_gather", "reduce_scatter", "all_to_all"]


def _sig(l, name, res, args):
    f = getattr(l, name)
    f.restype = res
    f.argtypes = args


def lib():
    """Loads libseqplan_isp.so (building it if absent). Raises if it cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists() or os.environ.get("SEQPLAN_ISP_REBUILD"):
        from .build import build
        build()
    l = ctypes.CDLL(str(_LIB_PATH), mode=ctypes.RTLD_GLOBAL)
    P = ctypes.POINTER
    _sig(l, "seqplan_isp_debug_gemm", c_int,
         [c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_int, c_int, c_int, c_vp,
          c_i64, c_vp, c_i64, c_vp, c_f, c_int, c_int, c_vp])
    for name, res, args in _EXTRA_SIGS:
        _sig(l, name, res, args)
    _lib = l
    return l


P = ctypes.POINTER
_EXTRA_SIGS = [
    ("seqplan_isp_ctx_create", c_int, [c_int, c_int, c_int, P(ShapeC), P(StrategyC), P(PolicyC),
                                       c_u32, P(c_vp)]),
    ("seqplan_isp_ctx_destroy", None, [c_vp]),
    ("seqplan_isp_last_error", ctypes.c_char_p, [c_vp]),
    ("seqplan_isp_ipc_handle_size", ctypes.c_size_t, []),
    ("seqplan_isp_ipc_handle", c_int, [c_vp, c_vp]),
    ("seqplan_isp_open_peers", c_int, [c_vp, c_vp]),
    ("seqplan_isp_nvls_export", c_int, [c_vp, P(c_int), P(c_int)]),
    ("seqplan_isp_nvls_attach", c_int, [c_vp, c_int, c_int]),
    ("seqplan_isp_nvls_bind", c_int, [c_vp]),
    ("seqplan_isp_nvls_release", c_int, [c_vp]),
    ("seqplan_isp_nvls_active", c_int, [c_vp]),
    ("seqplan_isp_group_create", c_int, [c_int, c_int, P(ShapeC), P(PolicyC), c_u32, P(c_vp)]),
    ("seqplan_isp_group_fwd", c_int, [P(c_vp), c_int, P(c_vp), P(c_vp), c_vp]),
    ("seqplan_isp_group_bwd", c_int, [P(c_vp), c_int, P(c_vp), P(c_vp), c_vp]),
    ("seqplan_isp_init_weights", c_int, [c_vp, c_u64]),
    ("seqplan_isp_shard_numel", c_i64, [c_vp, c_int]),
    ("seqplan_isp_set_weight_shard", c_int, [c_vp, c_int, c_vp, c_i64]),
    ("seqplan_isp_get_weight_shard", c_int, [c_vp, c_int, c_vp, c_i64]),
    ("seqplan_isp_get_grad_shard", c_int, [c_vp, c_int, c_vp, c_i64]),
    ("seqplan_isp_grad_shard_ptr", c_int, [c_vp, c_int, P(c_vp)]),
    ("seqplan_isp_fill_activation", c_int, [c_vp, c_u64, c_int, c_vp, c_vp]),
    ("seqplan_isp_block_fwd", c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("seqplan_isp_block_bwd", c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("seqplan_isp_pool_stats", c_int, [c_vp, P(StepStatsC)]),
    ("seqplan_isp_pool_replay", c_int, [c_vp, P(StepStatsC), P(c_i64)]),
    ("seqplan_isp_timeline", c_int, [c_vp, P(EventC), P(c_i64)]),
    ("seqplan_isp_kernel_profile", c_int, [c_vp, P(KernelRecC), P(c_i64), c_int]),
    ("seqplan_isp_launch_count", c_i64, [c_vp]),
    ("seqplan_isp_adamw_step", c_int, [c_vp, P(AdamWC), c_vp]),
    ("seqplan_isp_stack_create", c_int, [c_int, c_int, c_int, c_int, P(ShapeC), P(StrategyC), P(PolicyC), c_u32,
                                         P(c_vp)]),
    ("seqplan_isp_stack_destroy", None, [c_vp]),
    ("seqplan_isp_stack_layers", c_int, [c_vp]),
    ("seqplan_isp_stack_layer", c_vp, [c_vp, c_int]),
    ("seqplan_isp_stack_fwd", c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("seqplan_isp_stack_bwd", c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("seqplan_isp_debug_gather_bench", c_int, [c_vp, c_int, c_int, P(ctypes.c_float)]),
    ("seqplan_isp_debug_attention", c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_int, c_int, c_int,
                                            c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    ("seqplan_isp_debug_attention_ws", c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_int, c_int, c_int,
                                               c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    ("seqplan_isp_debug_attention_ds_bytes", c_i64, [c_int]),
    ("seqplan_isp_debug_rmsnorm", c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_f,
                                          c_vp]),
    ("seqplan_isp_link_local_peers", c_int, [P(c_vp), c_int]),
    ("seqplan_isp_debug_all_to_all", c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, P(c_vp), c_vp, c_vp,
                                             c_vp, c_int, c_vp]),
    ("seqplan_isp_debug_reduce_scatter", c_int, [c_int, c_int, c_i64, P(c_vp), c_int, c_f, c_int, c_vp, c_vp]),
    ("seqplan_isp_debug_push_allgather", c_int, [c_int, c_int, P(c_vp), c_vp, c_i64, c_int, c_int, c_vp]),
]


def link_local_peers(blocks):
    """Links IspBlock ranks 0..p-1 created in this process on one device (no IPC): each runs the
    multi-process code path with its peers' heaps on the same GPU (include/seqplan_isp.h)."""
    arr = (c_vp * len(blocks))(*[b.h for b in blocks])
    check(lib().seqplan_isp_link_local_peers(arr, len(blocks)), None, "link_local_peers")


def check(status, ctx=None, what=""):
    if status != 0:
        msg = ""
        if ctx:
            m = lib().seqplan_isp_last_error(ctx)
            msg = m.decode() if m else ""
        raise RuntimeError(f"{what}: {STATUS.get(status, status)}: {msg}")


def debug_gemm(a, b, out, M, N, K, *, a_mn=False, b_mn=False, epi=0, resid=None, out2=None,
               out_b=None, scale=1.0, accumulate=False, interleave64=False, stream=0):
    """Kernel-level GEMM through the C ABI; tensors are torch CUDA tensors (plumbing)."""
    st = lib().seqplan_isp_debug_gemm(
        a.data_ptr(), a.stride(0), int(a_mn), b.data_ptr(), b.stride(0), int(b_mn),
        out.data_ptr(), out.stride(0), M, N, K, epi,
        resid.data_ptr() if resid is not None else None, resid.stride(0) if resid is not None else 0,
        out2.data_ptr() if out2 is not None else None, out2.stride(0) if out2 is not None else 0,
        out_b.data_ptr() if out_b is not None else None, float(scale), int(accumulate),
        int(interleave64), stream)
    check(st, what="debug_gemm")


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream_handle(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def make_shape(H, D, S, I=0, rope_base=10000.0, eps=1e-5):
    return ShapeC(H, D, S, I, rope_base, eps)


def make_policy(pinned=True, consolidate=0, premap=True, capacity=0):
    return PolicyC(int(pinned), consolidate, int(premap), capacity)


class IspBlock:
    """One rank's ISP block context (multi-process mode: one process per GPU).

    Thin ctypes wrapper; every call goes through the C ABI of include/seqplan_isp.h.
    """

    def __init__(self, H, D, S, world=1, rank=0, device=0, policy=None, flags=0, I=0, recompute=False,
                 micro_batches=1):
        l = lib()
        self.world, self.rank, self.device = world, rank, device
        self.shape = make_shape(H, D, S, I)
        # micro_batches = n (Strategy::micro_batch_num): n fwd/bwd calls per step, gradients accumulate
        strat = StrategyC(1, int(micro_batches), int(recompute), 1, 1, 1, world, world, 1, 1)
        pol = policy if policy is not None else make_policy()
        h = c_vp()
        st = l.seqplan_isp_ctx_create(world, rank, device, ctypes.byref(self.shape), ctypes.byref(strat),
                                      ctypes.byref(pol), flags, ctypes.byref(h))
        check(st, None, "seqplan_isp_ctx_create")
        self.h = h

    # -- peer bootstrap (world > 1) --
    def ipc_handle(self) -> bytes:
        n = lib().seqplan_isp_ipc_handle_size()
        buf = ctypes.create_string_buffer(n)
        check(lib().seqplan_isp_ipc_handle(self.h, buf), self.h, "ipc_handle")
        return buf.raw

    def open_peers(self, handles):
        blob = b"".join(handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        check(lib().seqplan_isp_open_peers(self.h, buf), self.h, "open_peers")

    # NVLink SHARP reduce-scatter setup (seqplan_isp_nvls_*; dist.bootstrap_nvls drives it)
    def nvls_export(self):
        """Rank 0: (pid, fd) of the exported multicast handle, or None when not applicable."""
        pid, fd = c_int(), c_int()
        r = lib().seqplan_isp_nvls_export(self.h, ctypes.byref(pid), ctypes.byref(fd))
        if r == ERR_UNSUPPORTED:
            return None
        check(r, self.h, "nvls_export")
        return pid.value, fd.value

    def nvls_attach(self, pid, fd) -> bool:
        return lib().seqplan_isp_nvls_attach(self.h, pid, fd) == 0

    def nvls_bind(self) -> bool:
        return lib().seqplan_isp_nvls_bind(self.h) == 0

    def nvls_release(self):
        lib().seqplan_isp_nvls_release(self.h)

    def nvls_active(self) -> bool:
        return bool(lib().seqplan_isp_nvls_active(self.h))

    def init_weights(self, seed):
        check(lib().seqplan_isp_init_weights(self.h, seed), self.h, "init_weights")

    def shard_numel(self, t):
        return lib().seqplan_isp_shard_numel(self.h, t)

    def set_weight_shard(self, t, arr):
        import numpy as np
        a = np.ascontiguousarray(arr, dtype=np.float32).reshape(-1)
        check(lib().seqplan_isp_set_weight_shard(self.h, t, a.ctypes.data, a.size), self.h, "set_weight_shard")

    def weight_shard(self, t):
        import numpy as np
        a = np.empty(self.shard_numel(t), np.float32)
        check(lib().seqplan_isp_get_weight_shard(self.h, t, a.ctypes.data, a.size), self.h, "get_weight_shard")
        return a

    def grad_shard(self, t):
        import numpy as np
        a = np.empty(self.shard_numel(t), np.float32)
        check(lib().seqplan_isp_get_grad_shard(self.h, t, a.ctypes.data, a.size), self.h, "get_grad_shard")
        return a

    def adamw_step(self, lr, step, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, stream=None):
        """AdamW on every fp32 master shard; refreshes the bf16 working shards."""
        p = AdamWC(lr, beta1, beta2, eps, weight_decay, step)
        check(lib().seqplan_isp_adamw_step(self.h, ctypes.byref(p), _stream_handle(stream)), self.h, "adamw_step")

    def fill_activation(self, seed, tid, out, stream=None):
        check(lib().seqplan_isp_fill_activation(self.h, seed, tid, out.data_ptr(), _stream_handle(stream)),
              self.h, "fill_activation")

    def fwd(self, x, y, stream=None):
        check(lib().seqplan_isp_block_fwd(self.h, x.data_ptr(), y.data_ptr(), _stream_handle(stream)),
              self.h, "block_fwd")

    def bwd(self, dy, dx, stream=None):
        check(lib().seqplan_isp_block_bwd(self.h, dy.data_ptr(), dx.data_ptr(), _stream_handle(stream)),
              self.h, "block_bwd")

    def pool_stats(self):
        s = StepStatsC()
        check(lib().seqplan_isp_pool_stats(self.h, ctypes.byref(s)), self.h, "pool_stats")
        return {n: getattr(s, n) for n, _ in StepStatsC._fields_}

    def pool_replay(self):
        """run_mempool (mempool.hpp:285-387) over the device pool's own recorded trace."""
        s = StepStatsC()
        n = c_i64(0)
        check(lib().seqplan_isp_pool_replay(self.h, ctypes.byref(s), ctypes.byref(n)), self.h, "pool_replay")
        d = {k: getattr(s, k) for k, _ in StepStatsC._fields_}
        d["trace_ops"] = n.value
        return d

    def timeline(self):
        n = c_i64(0)
        lib().seqplan_isp_timeline(self.h, None, ctypes.byref(n))
        arr = (EventC * max(n.value, 1))()
        lib().seqplan_isp_timeline(self.h, arr, ctypes.byref(n))
        return [dict(stream=e.stream, kind=EV_NAMES[e.kind], layer=e.layer, start=e.start_s, end=e.end_s)
                for e in arr[:n.value]]

    def kernel_profile(self, clear=True):
        n = c_i64(0)
        lib().seqplan_isp_kernel_profile(self.h, None, ctypes.byref(n), 0)
        arr = (KernelRecC * max(n.value, 1))()
        lib().seqplan_isp_kernel_profile(self.h, arr, ctypes.byref(n), int(clear))
        return [dict(kind=K_NAMES[r.kind], flops=r.flops, bytes=r.bytes, seconds=r.seconds) for r in arr[:n.value]]

    def launch_count(self):
        return lib().seqplan_isp_launch_count(self.h)

    def close(self):
        if getattr(self, "h", None) and getattr(self, "_owner", True):
            lib().seqplan_isp_ctx_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class IspStack:
    """`layers` ISP blocks run as one step: inter-layer prefetch of every
    layer's gathers on one comm stream; layer(l) is a non-owning IspBlock view (weights, grads,
    peer bootstrap, timeline of that layer)."""

    def __init__(self, layers, H, D, S, world=1, rank=0, device=0, policy=None, flags=0, I=0, recompute=False):
        l = lib()
        self.world, self.rank = world, rank
        self.shape = make_shape(H, D, S, I)
        strat = StrategyC(1, 1, int(recompute), 1, 1, 1, world, world, 1, 1)
        pol = policy if policy is not None else make_policy()
        h = c_vp()
        check(l.seqplan_isp_stack_create(layers, world, rank, device, ctypes.byref(self.shape), ctypes.byref(strat),
                                         ctypes.byref(pol), flags, ctypes.byref(h)), None, "stack_create")
        self.h = h
        self.n = layers

    def layer(self, i):
        b = IspBlock.__new__(IspBlock)
        b.h, b.world, b.rank, b.shape = c_vp(lib().seqplan_isp_stack_layer(self.h, i)), self.world, self.rank, self.shape
        b._owner = False  # a view: the stack owns and destroys the context
        return b

    def fwd(self, x, y, stream=None):
        check(lib().seqplan_isp_stack_fwd(self.h, x.data_ptr(), y.data_ptr(), _stream_handle(stream)),
              self.layer(0).h, "stack_fwd")

    def bwd(self, dy, dx, stream=None):
        check(lib().seqplan_isp_stack_bwd(self.h, dy.data_ptr(), dx.data_ptr(), _stream_handle(stream)),
              self.layer(0).h, "stack_bwd")

    def close(self):
        if getattr(self, "h", None):
            lib().seqplan_isp_stack_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class IspGroup:
    """p ranks on one GPU in one process (lock-step phases; tests and single-GPU parity)."""

    def __init__(self, H, D, S, world, device=0, policy=None, flags=0, I=0):
        l = lib()
        self.world = world
        self.shape = make_shape(H, D, S, I)
        pol = policy if policy is not None else make_policy()
        arr = (c_vp * world)()
        check(l.seqplan_isp_group_create(world, device, ctypes.byref(self.shape), ctypes.byref(pol), flags, arr),
              None, "group_create")
        self.hs = [c_vp(arr[i]) for i in range(world)]
        self._arr = arr

    def rank(self, r):
        b = IspBlock.__new__(IspBlock)
        b.h, b.world, b.rank, b.shape = self.hs[r], self.world, r, self.shape
        b._owner = False  # a view: the group owns and destroys the context
        return b

    def fwd(self, xs, ys, stream=None):
        X = (c_vp * self.world)(*[x.data_ptr() for x in xs])
        Y = (c_vp * self.world)(*[y.data_ptr() for y in ys])
        check(lib().seqplan_isp_group_fwd(self._arr, self.world, X, Y, _stream_handle(stream)), self.hs[0], "group_fwd")

    def bwd(self, dys, dxs, stream=None):
        X = (c_vp * self.world)(*[x.data_ptr() for x in dys])
        Y = (c_vp * self.world)(*[y.data_ptr() for y in dxs])
        check(lib().seqplan_isp_group_bwd(self._arr, self.world, X, Y, _stream_handle(stream)), self.hs[0], "group_bwd")

    def close(self):
        if getattr(self, "hs", None):
            for h in self.hs:
                lib().seqplan_isp_ctx_destroy(h)
            self.hs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
