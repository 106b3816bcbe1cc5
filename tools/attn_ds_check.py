"""Development: stored-dS backward (key-tile kernel + dQ kernel) against the two-role kernel —
outputs compared and both timed (CUDA events); not the bench contract."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_09149_b200 import capi  # noqa: E402


def run(S, heads, ws_gb, iters=5):
    dev = torch.device("cuda")
    d = 128
    Hl = heads * d
    torch.manual_seed(0)
    qkv = torch.randn(S, 3 * Hl, device=dev).bfloat16()
    o = torch.empty(S, Hl, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(heads, S, device=dev)
    do = torch.randn(S, Hl, device=dev).bfloat16()
    delta = torch.empty(heads, S, device=dev)
    dq_acc = torch.empty(heads * S * d, device=dev)
    per_head = capi.lib().seqplan_isp_debug_attention_ds_bytes(S)
    ws_bytes = min(int(ws_gb * (1 << 30)), per_head * heads)
    ws = torch.empty(ws_bytes, device=dev, dtype=torch.uint8)
    l = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    q, k, v = qkv.data_ptr(), qkv[:, Hl:].data_ptr(), qkv[:, 2 * Hl:].data_ptr()
    capi.check(l.seqplan_isp_debug_attention(q, k, v, 3 * Hl, o.data_ptr(), Hl, lse.data_ptr(), S, heads, d,
                                             None, None, None, None, 0, None, None, st))
    outs = {}
    for name, wsp, wsb in (("split", None, 0), ("ds", ws.data_ptr(), ws_bytes)):
        dqkv = torch.zeros_like(qkv)

        def bw():
            capi.check(l.seqplan_isp_debug_attention_ws(q, k, v, 3 * Hl, o.data_ptr(), Hl, lse.data_ptr(), S, heads,
                                                        d, do.data_ptr(), dqkv.data_ptr(), dqkv[:, Hl:].data_ptr(),
                                                        dqkv[:, 2 * Hl:].data_ptr(), 3 * Hl, delta.data_ptr(),
                                                        dq_acc.data_ptr(), wsp, wsb, st))
        bw(); torch.cuda.synchronize()
        outs[name] = dqkv.clone()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            bw()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        print(f"S={S} heads={heads} {name} ws={wsb / 2**30:.2f} GiB: bwd {ms:.3f} ms {4.0 * S * S * Hl / ms / 1e9:.0f} TF/s",
              flush=True)
    a, b = outs["split"].float(), outs["ds"].float()
    for i, nm in enumerate("qkv"):
        x, y = a[:, i * Hl:(i + 1) * Hl], b[:, i * Hl:(i + 1) * Hl]
        rel = ((x - y).norm() / x.norm()).item()
        print(f"  d{nm}: rel-L2 {rel:.3e} max|diff| {(x - y).abs().max().item():.3e} equal {torch.equal(x, y)}")


if __name__ == "__main__":
    cfgs = [(16384, 16, 64), (32768, 32, 64), (32768, 32, 8), (4096, 32, 8)]
    if len(sys.argv) > 1:
        cfgs = [tuple(float(x) if i == 2 else int(x) for i, x in enumerate(a.split(","))) for a in sys.argv[1:]]
    for S, h, g in cfgs:
        run(S, h, g)
