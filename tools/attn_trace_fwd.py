"""clock64 trace of the production attention forward (CTA 0, head 0): per key tile j, the time
the MMA warp issued PV_A(j) / PV_B(j) and, per stream, when softmax got S_x(j) and when it
released P_x(j). Development tool (reads the debug trace hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_09149_b200 import capi
from tools.attn_bench import run
l = capi.lib()
buf = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
l.seqplan_isp_debug_set_trace_fwd.argtypes = [ctypes.c_void_p]
l.seqplan_isp_debug_set_trace_fwd(buf.data_ptr())
run(int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 16, 128, iters=1, bwd=False)
t = buf.view(64, 8).cpu().tolist()
base = t[0][4]
print("j | MMA: pA_ok PV_A pB_ok PV_B | CTA0 A p_done quads 0..3")
for j in range(40):
    r = t[j]
    if r[4] == 0: break
    f = lambda x: x - base if x else -1
    print(j, [f(v) for v in r[0:4]], [f(v) for v in r[4:8]])
