"""Development timing of the attention kernels (CUDA events); not the bench contract."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_09149_b200 import capi


def run(S, heads, d, bwd=True, iters=5):
    dev = torch.device("cuda")
    Hl = heads * d
    qkv = torch.randn(S, 3 * Hl, device=dev).bfloat16()
    o = torch.empty(S, Hl, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(heads, S, device=dev)
    do = torch.randn(S, Hl, device=dev).bfloat16()
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(heads, S, device=dev)
    dq_acc = torch.empty(heads * S * d, device=dev)
    l = capi.lib()
    # the block's default backward: the stored-dS pair with every head's dS tiles in one workspace
    # (ATTN_BENCH_SPLIT=1: the two-role kernel)
    nws = 0 if os.environ.get("ATTN_BENCH_SPLIT") or d != 128 else l.seqplan_isp_debug_attention_ds_bytes(S) * heads
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    q, k, v = qkv.data_ptr(), qkv[:, Hl:].data_ptr(), qkv[:, 2 * Hl:].data_ptr()

    def fwd():
        capi.check(l.seqplan_isp_debug_attention(q, k, v, 3 * Hl, o.data_ptr(), Hl, lse.data_ptr(), S, heads, d,
                                                 None, None, None, None, 0, None, None, st))

    def bw():
        capi.check(l.seqplan_isp_debug_attention_ws(q, k, v, 3 * Hl, o.data_ptr(), Hl, lse.data_ptr(), S, heads, d,
                                                    do.data_ptr(), dqkv.data_ptr(), dqkv[:, Hl:].data_ptr(),
                                                    dqkv[:, 2 * Hl:].data_ptr(), 3 * Hl, delta.data_ptr(),
                                                    dq_acc.data_ptr(), ws.data_ptr() if nws else None, nws, st))
    out = []
    for name, fn, mult in (("fwd", fwd, 2.0), ("bwd", bw, 4.0)):
        if name == "bwd" and not bwd:
            continue
        fn(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        tf = mult * S * S * Hl / ms / 1e9
        out.append(f"{name} {ms:.3f} ms {tf:.0f} TF/s")
    print(f"S={S} heads={heads} d={d}: " + " | ".join(out), flush=True)


if __name__ == "__main__":
    for S, h, d in [(4096, 32, 128), (16384, 16, 128), (32768, 16, 128), (4096, 8, 64)]:
        run(S, h, d)
