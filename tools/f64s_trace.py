"""Per-sweep behaviour of the CNTGW_F64S plan on the C5 law: for each sweep of
one loop (after `outer` outer steps), the f- and g-update kernel times
(CUDA events), whether the sweep measured, and the kept fraction of the
(row group, stage) pairs."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import configs, engine, solvers
from paper_2602_06658_b200._native import F64S, call

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 60
law = sys.argv[4] if len(sys.argv) > 4 else "c5"
torch.cuda.set_device(0)
os.environ["CNTGW_PRECISION"] = "f64s"
pc = configs.GENERATORS[law.upper()](seed=0, n=n)
EPS = configs.C5_EPS if law == "c5" else configs.C4_EPS
src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=pc.x.shape[1])
tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=pc.y.shape[1])
st = solvers._CntGwState(src, tgt, P.make_config(EPS, n_inner=50, max_outer=outer + 1))
for _ in range(outer):
    st.step()
dev = st.dev
dev.set_gamma(st.gamma)
dev.choose_precision(st.f, st.g, EPS / 8)
eps = EPS / 8
loop = dev.loop
loop.state.init(eps, None, None, sweeps + 5, "symmetrized")
out = torch.zeros(3, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def dens(op):
    call("cntgw_f64s_plan_density", op.kd, 1, op.rows.n, op.cols.n, op.ws.data_ptr(), out.data_ptr(), s)
    o = out.cpu().numpy()
    return o[0] / o[1], int(o[2])
for k in range(1, sweeps + 1):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    loop.state.begin()
    e[0].record()
    dev.fwd(loop.state, st.g, loop.ft)
    e[1].record()
    dev.bwd(loop.state, st.f, loop.gt)
    e[2].record()
    torch.cuda.synchronize()
    df, mf = dens(dev.fwd)
    dg, mg = dens(dev.bwd)
    print(f"sweep {k}: f {e[0].elapsed_time(e[1]):7.1f} ms measured={mf} kept={df:.4f} | "
          f"g {e[1].elapsed_time(e[2]):7.1f} ms measured={mg} kept={dg:.4f}", flush=True)
    call("cntgw_sweep_apply", loop.state.ptr, st.f.data_ptr(), loop.ft.data_ptr(), dev.n, 1, s)
    call("cntgw_sweep_apply", loop.state.ptr, st.g.data_ptr(), loop.gt.data_ptr(), dev.m, 1, s)
