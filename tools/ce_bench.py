"""Copy-engine peer bandwidth microbenchmark (2+ GPUs, one process): single copy, concurrent
copies from several streams, and 2-D strided copies like the gate|up gather."""
import torch

n = torch.cuda.device_count()
assert n >= 2
MB = 1 << 20
for size in (16 * MB, 64 * MB, 256 * MB):
    src = torch.empty(size, dtype=torch.uint8, device="cuda:1")
    dst = torch.empty(size, dtype=torch.uint8, device="cuda:0")
    torch.cuda.set_device(0)
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        dst.copy_(src, non_blocking=True)
    e.record(); torch.cuda.synchronize(0)
    print(f"pull {size/MB:.0f} MB: {10*size/(s.elapsed_time(e)/1e3)/1e9:.0f} GB/s", flush=True)
# concurrent pulls from all peers into device 0
size = 128 * MB
torch.cuda.set_device(0)
srcs = [torch.empty(size, dtype=torch.uint8, device=f"cuda:{q}") for q in range(1, n)]
dsts = [torch.empty(size, dtype=torch.uint8, device="cuda:0") for _ in range(1, n)]
streams = [torch.cuda.Stream(device=0) for _ in range(1, n)]
for _ in range(2):
    for st, d, s_ in zip(streams, dsts, srcs):
        with torch.cuda.stream(st):
            d.copy_(s_, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for st in streams:
    st.wait_event(s)
for _ in range(5):
    for st, d, s_ in zip(streams, dsts, srcs):
        with torch.cuda.stream(st):
            d.copy_(s_, non_blocking=True)
for st in streams:
    e2 = torch.cuda.Event(); e2.record(st); torch.cuda.current_stream(0).wait_event(e2)
e.record(); torch.cuda.synchronize()
print(f"concurrent pulls from {n-1} peers: {5*(n-1)*size/(s.elapsed_time(e)/1e3)/1e9:.0f} GB/s total", flush=True)
# local D2D
a = torch.empty(256 * MB, dtype=torch.uint8, device="cuda:0"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize(); s.record()
for _ in range(10): b.copy_(a)
e.record(); torch.cuda.synchronize()
print(f"local D2D 256MB: {10*256*MB/(s.elapsed_time(e)/1e3)/1e9:.0f} GB/s (read) ", flush=True)
