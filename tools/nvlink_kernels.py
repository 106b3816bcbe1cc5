"""NVLink evidence for the ISP collective kernels.

One process drives GPU 0 as rank 0 of p ranks (p = visible GPUs, at most 4) with peer access to
the others, and runs the library's own collective kernels at the 7B-32K per-rank sizes through the
C ABI: the Ulysses all-to-all pulls (token->head for q|k|v, head->token for dq|dk|dv), the
gradient reduce-scatter pull (fixed-rank-order fp32 sum, fused cast/scale), and the push
all-gather of a weight shard (vector-store and cp.async.bulk variants). Each line: CUDA-event time,
the bytes that cross NVLink into or out of GPU 0 ((p-1)/p of the exchanged data), GB/s vs the
900 GB/s nominal and 770 GB/s measured peer-copy bandwidth (B200_PROFILING.md). Under
`ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,...` (single process, kernels replay-safe) the
same run gives the counted link bytes per kernel.

    python tools/nvlink_kernels.py [iters]
    python tools/nvlink_kernels.py --vpro profiles/r2/vpro_kernels_p<N>.csv   # message-size sweep
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_09149_b200 import capi  # noqa: E402

H, S, D = 4096, 32768, 32


def enable_peers(p):
    rt = ctypes.CDLL("libcudart.so.12")
    for a in range(p):
        rt.cudaSetDevice(a)
        for b in range(p):
            if a != b:
                rc = rt.cudaDeviceEnablePeerAccess(b, 0)
                assert rc in (0, 704), rc  # 704: already enabled
    rt.cudaSetDevice(0)


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    p = min(torch.cuda.device_count(), 4)
    assert p >= 2, "needs >= 2 GPUs"
    enable_peers(p)
    l = capi.lib()
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream(0).cuda_stream
    T, Hl = S // p, H // p
    frac = (p - 1) / p
    rows = []

    def report(name, sec, remote_bytes, note):
        gbs = remote_bytes / sec / 1e9
        rows.append({"kernel": name, "p": p, "ms": sec * 1e3, "nvlink_bytes": remote_bytes, "gb_s": gbs,
                     "frac_of_900": gbs / 900.0, "frac_of_770": gbs / 770.0, "note": note})
        print(json.dumps(rows[-1]), flush=True)

    # all-to-all tokens -> heads (q|k|v): rank q's [T, 3H] token rows, this rank's heads [S, 3Hl]
    tok = [torch.randn(T, 3 * H, device=f"cuda:{q}").bfloat16() for q in range(p)]
    dst = torch.empty(S, 3 * Hl, device="cuda:0", dtype=torch.bfloat16)
    sec = timed(lambda: capi.check(l.seqplan_isp_debug_all_to_all(p, 0, T, H, 3, 128, +1, ptrs(tok), dst.data_ptr(),
                                                                  None, None, 0, st)), iters)
    report("a2a_to_heads_kernel (q|k|v)", sec, frac * S * 3 * Hl * 2, "pull: reads (p-1)/p of its [S, 3H/p] rows from peers")
    # all-to-all heads -> tokens (dq|dk|dv)
    heads = [torch.randn(S, 3 * Hl, device=f"cuda:{q}").bfloat16() for q in range(p)]
    back = torch.empty(T, 3 * H, device="cuda:0", dtype=torch.bfloat16)
    sec = timed(lambda: capi.check(l.seqplan_isp_debug_all_to_all(p, 0, T, H, 3, 128, -1, ptrs(heads), back.data_ptr(),
                                                                  None, None, 0, st)), iters)
    report("a2a_to_tokens_kernel (dq|dk|dv)", sec, frac * T * 3 * H * 2, "pull")
    del tok, heads, dst, back
    # reduce-scatter of the QKV weight-gradient partial (bf16 [3H, H] on every rank)
    n = 3 * H * H
    part = [torch.randn(n, device=f"cuda:{q}").bfloat16() for q in range(p)]
    out = torch.zeros(n // p, device="cuda:0")
    sec = timed(lambda: capi.check(l.seqplan_isp_debug_reduce_scatter(p, 0, n // p, ptrs(part), 0, 1.0, 0,
                                                                      out.data_ptr(), st)), iters)
    report("reduce_scatter_kernel<bf16> (QKV grad)", sec, frac * n * 2, "pull of this rank's slice from every peer")
    del part, out
    # push all-gather of the QKV weight shard into every rank's gathered buffer
    shard = torch.randn(n // p, device="cuda:0").bfloat16()
    gath = [torch.empty(n, device=f"cuda:{q}", dtype=torch.bfloat16) for q in range(p)]
    for kind, name, ctas in ((1, "push_bulk_kernel<16KB,2> (QKV weight AG)", 96), (0, "push_copy_kernel (QKV weight AG)", 148)):
        sec = timed(lambda: capi.check(l.seqplan_isp_debug_push_allgather(p, 0, ptrs(gath), shard.data_ptr(),
                                                                          n // p * 2, kind, ctas, st)), iters)
        report(name, sec, (p - 1) * n // p * 2, "push: this rank's shard stored into every peer")
    print(json.dumps({"summary": rows}), flush=True)


def vpro(out_csv, iters=5):
    """Measured VPro curves in the reference's CSV schema (bandwidth.hpp:214-253): the library's
    all-gather (push, bulk-copy), reduce-scatter (pull, fp32 sum + cast) and all-to-all (pull)
    kernels of rank 0 at full-tensor message sizes 4..256 MiB in the tau convention of cost.hpp:177-188
    (bandwidth = message bytes / time). Rows for both axes ("intra", "inter": one NVSwitch box, the
    placement's inter label for sp = ps = p)."""
    p = min(torch.cuda.device_count(), 4)
    enable_peers(p)
    l = capi.lib()
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream(0).cuda_stream
    rows = []
    for mib in (4, 16, 64, 256):
        v = mib << 20
        # all-gather: each rank contributes v / p bytes of a v-byte tensor
        shard = torch.empty(v // p // 2, device="cuda:0", dtype=torch.bfloat16)
        gath = [torch.empty(v // 2, device=f"cuda:{q}", dtype=torch.bfloat16) for q in range(p)]
        t = timed(lambda: capi.check(l.seqplan_isp_debug_push_allgather(p, 0, ptrs(gath), shard.data_ptr(), v // p,
                                                                        1, 96, st)), iters)
        rows.append(("all-gather", p, v, v / t))
        del shard, gath
        # reduce-scatter of a v-byte bf16 partial
        part = [torch.empty(v // 2, device=f"cuda:{q}", dtype=torch.bfloat16).normal_() for q in range(p)]
        out = torch.empty(v // 2 // p, device="cuda:0")
        t = timed(lambda: capi.check(l.seqplan_isp_debug_reduce_scatter(p, 0, v // 2 // p, ptrs(part), 0, 1.0, 0,
                                                                        out.data_ptr(), st)), iters)
        rows.append(("reduce-scatter", p, v, v / t))
        del part, out
        # all-to-all of a v-byte [S, 3H] activation (H = 4096): T = v / (p * 3H * 2) rows per rank
        Tq = max(8, v // (p * 3 * H * 2))
        tok = [torch.empty(Tq, 3 * H, device=f"cuda:{q}", dtype=torch.bfloat16) for q in range(p)]
        dst = torch.empty(p * Tq, 3 * (H // p), device="cuda:0", dtype=torch.bfloat16)
        t = timed(lambda: capi.check(l.seqplan_isp_debug_all_to_all(p, 0, Tq, H, 3, 128, +1, ptrs(tok), dst.data_ptr(),
                                                                    None, None, 0, st)), iters)
        rows.append(("all-to-all", p, p * Tq * 3 * H * 2, p * Tq * 3 * H * 2 / t))
        del tok, dst
    with open(out_csv, "w") as f:
        f.write("# measured on B200 by tools/nvlink_kernels.py --vpro (rank-0 kernel, CUDA events, isolated)\n")
        f.write("op,participants,axis,message_bytes,bandwidth_bytes_per_sec\n")
        for op, n, v, bw in rows:
            for axis in ("intra", "inter"):
                f.write(f"{op},{n},{axis},{v},{bw:.6e}\n")
    print(json.dumps({"vpro": out_csv, "rows": len(rows)}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--vpro":
        vpro(sys.argv[2])
    else:
        main()
