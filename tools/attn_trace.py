import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_09149_b200 import capi
from tools.attn_bench import run
l = capi.lib()
buf = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
l.seqplan_isp_debug_set_trace.argtypes = [ctypes.c_void_p]
l.seqplan_isp_debug_set_trace(buf.data_ptr())
run(8192, 16, 128, iters=1)
t = buf.view(64, 8).cpu().tolist()
base = t[0][0]
print("i | S_issued grads_issued | c:start s_full_ok p_wait_start p_free_ok done")
prev = None
for i, r in enumerate(t[:40]):
    if r[0] == 0: break
    v = [x - base if x else -1 for x in r[:7]]
    print(i, v, "per-iter", (r[6] - prev) if prev else None)
    prev = r[6]
