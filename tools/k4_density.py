"""Kept fraction of the F64S plan as the K4 plan pass voted it (after each
outer step), and the K4 kernel time: python tools/k4_density.py [c4|c5] [n] [steps]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import configs, solvers
from paper_2602_06658_b200._native import call

law = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 20 if law == "c4" else 1 << 18)
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
torch.cuda.set_device(0)
pc = configs.GENERATORS[law.upper()](seed=0, n=n)
eps, inner = (configs.C4_EPS, 100) if law == "c4" else (configs.C5_EPS, 200)
src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=pc.x.shape[1])
tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=pc.y.shape[1])
st = solvers._CntGwState(src, tgt, P.make_config(eps, n_inner=inner, max_outer=steps))
out = torch.zeros(3, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for k in range(steps):
    st.step()
    dev = st.dev
    op = dev.fwd
    call("cntgw_f64s_plan_density", op.kd, 1, op.rows.n, op.cols.n, op.ws.data_ptr(), out.data_ptr(), s)
    o = out.cpu().numpy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.plan_pass(st.f, st.g)
    e1.record()
    torch.cuda.synchronize()
    print(f"step {k + 1}: K4 kept {o[0] / o[1]:.4f} of the (group, stage) pairs, flags {int(o[2])}, "
          f"plan pass {e0.elapsed_time(e1):.1f} ms", flush=True)
