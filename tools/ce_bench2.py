"""Copy-engine concurrency: k streams each pulling 16/32 MB chunks from the same peer."""
import torch
MB = 1 << 20
torch.cuda.set_device(0)
for size in (8 * MB, 16 * MB, 32 * MB):
    for k in (1, 2, 4, 8):
        srcs = [torch.empty(size, dtype=torch.uint8, device="cuda:1") for _ in range(k)]
        dsts = [torch.empty(size, dtype=torch.uint8, device="cuda:0") for _ in range(k)]
        sts = [torch.cuda.Stream(device=0) for _ in range(k)]
        def go(it):
            for _ in range(it):
                for st, d, s_ in zip(sts, dsts, srcs):
                    with torch.cuda.stream(st):
                        d.copy_(s_, non_blocking=True)
        go(2); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for st in sts: st.wait_event(s)
        go(8)
        for st in sts:
            ev = torch.cuda.Event(); ev.record(st); torch.cuda.current_stream().wait_event(ev)
        e.record(); torch.cuda.synchronize()
        print(f"{size//MB} MB x {k} streams: {8*k*size/(s.elapsed_time(e)/1e3)/1e9:.0f} GB/s", flush=True)
