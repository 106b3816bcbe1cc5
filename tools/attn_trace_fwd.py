import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_09149_b200 import capi
from tools.attn_bench import run
l = capi.lib()
buf = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
l.seqplan_isp_debug_set_trace_fwd.argtypes = [ctypes.c_void_p]
l.seqplan_isp_debug_set_trace_fwd(buf.data_ptr())
run(8192, 16, 128, iters=1)
t = buf.view(64, 8).cpu().tolist()
base = t[0][0]
print("j | S_issued PV_issued | sm:wait_s s_ok xchg_ok exp_done arrived")
prev = None
for i, r in enumerate(t[:40]):
    if r[0] == 0: break
    v = [x - base if x else -1 for x in r[:7]]
    print(i, v, "per-tile", (r[6] - prev) if prev else None)
    prev = r[6]
