import sys, numpy as np, torch
sys.path.insert(0, '.')
import importlib
import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import engine, configs
S = importlib.import_module("paper_2602_06658_b200.sinkhorn")
from oracle import cntgw_oracle as O
dev = torch.device('cuda', 0)
for (n, m, k) in [(128, 256, 16), (129, 257, 16), (1000, 1000, 8), (4096, 4096, 16)]:
    inst = configs.c2(seed=1, n=n, m=m, k=k)
    a, b = np.full(n, 1/n), np.full(m, 1/m)
    cost = P.SeparableLowRankCost(inst.u, inst.v, inst.row_sep, inst.col_sep)
    prob = S.device_problem(cost, a, b, dev)
    want = O.softmin(O.LowRank(inst.u, inst.v, inst.row_sep, inst.col_sep), np.log(b), inst.g.astype(float), inst.eps)
    for prec in (0, 2):
        prob.fwd.prec = prec
        st = engine.SweepState(dev); st.init(inst.eps)
        gt = engine.to_dev64(inst.g.astype(float) - prob.col_sep, dev)
        out = torch.empty(n, dtype=torch.float64, device=dev)
        prob.fwd(st, gt, out, skip=False)
        torch.cuda.synchronize()
        got = out.cpu().numpy() + prob.row_sep
        print(n, m, k, prec, np.abs(got - want).max() / np.abs(want).max(), got[:3], want[:3], flush=True)
