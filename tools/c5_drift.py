"""Per-sweep drift of the column records on the C5 law (design probe for the
CNTGW_F64S plan margin): after `outer` outer steps, run sweeps one at a time
and print lam * max_j |g~_j(new) - g~_j(old)| (f-update records) and the
same for f~ (g-update records), plus the needed (row group, stage) fraction
of the f-update at several thresholds T (natural order)."""
import math, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import configs, engine, solvers
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from c5_sparsity import need_fraction

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 1
torch.cuda.set_device(0)
os.environ["CNTGW_PRECISION"] = "f64"
pc = configs.c5(seed=0, n=n)
src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=64)
tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=32)
st = solvers._CntGwState(src, tgt, P.make_config(configs.C5_EPS, n_inner=200, max_outer=outer + 1))
for k in range(outer):
    st.step()
dev = st.dev
dev.set_gamma(st.gamma)
dev.choose_precision(st.f, st.g, configs.C5_EPS / 8)
eps = configs.C5_EPS / 8
lam = math.log2(math.e) / eps
loop = dev.loop
loop.state.init(eps, None, None, 400, "symmetrized")
for s in range(1, 201):
    f0, g0 = st.f.clone(), st.g.clone()
    loop.sweep(st.f, st.g, "symmetrized")
    if s in (1, 2, 3, 5, 10, 20, 50, 100, 150, 200):
        dg = float((st.g - g0).abs().max()) * lam
        df = float((st.f - f0).abs().max()) * lam
        dg99 = float(torch.quantile((st.g - g0).abs()[:1 << 16], 0.99)) * lam
        print(f"sweep {s}: lam max|dg| {dg:.3e} (p99 {dg99:.3e})  lam max|df| {df:.3e}", flush=True)
xr, zc, sr, tc = dev.src.feat64, dev.tgt.feat64, dev.sx, dev.ty
g, lb = st.g, dev.tgt.log2w
def q_rows(rows, cols):
    x, s_ = xr[rows], sr[rows]
    z, t = zc[cols], tc[cols]
    return -(lam * (g[cols][None, :] + 2.0 * (x @ z.t()) - (s_[:, None] - t[None, :]) ** 2) + lb[cols][None, :])
nat_r = torch.arange(dev.n, device=xr.device)
nat_c = torch.arange(dev.m, device=xr.device)
for T in (64.0, 1024.0, 8192.0, 65536.0, 5e5):
    print(f"T={T:.0f}: natural needed fraction {need_fraction(q_rows, nat_r, nat_c, T):.4f}; "
          f"cluster order {need_fraction(q_rows, dev.src.locality(), dev.tgt.locality(), T):.4f}", flush=True)
