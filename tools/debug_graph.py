import sys, os
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import solvers
g = dict(np.load('tests/golden/c1_solve.npz'))
src = P.EmbeddedMeasure(g['x_feat'], g['a']); tgt = P.EmbeddedMeasure(g['y_feat'], g['b'])
for kw in (dict(n_inner=5, max_outer=1), dict(n_inner=5, max_outer=3), dict(threshold=1e-5, max_inner=200, max_outer=2)):
    cfg = P.make_config(0.01, **kw)
    st = solvers._CntGwState(src, tgt, cfg)
    ds = solvers._DeviceSolve(st)
    rows, conv, err = ds.run()
    print(kw, rows, conv, err, flush=True)
    print('  f finite', torch.isfinite(st.f).all().item(), st.f[:3].tolist(), 'g', st.g[:3].tolist(), flush=True)
    print('  state', st.dev.loop.state.read().applied, st.dev.loop.state.read().eps_n, flush=True)
    os.environ['CNTGW_DEVICE_LOOP'] = '0'
    res = P.solve_cnt_gw(src, tgt, cfg) if 'threshold' in kw else None
    st2 = solvers._CntGwState(src, tgt, cfg)
    s2 = st2.step()
    print('  host step1', s2, st2.f[:3].tolist(), flush=True)
    os.environ['CNTGW_DEVICE_LOOP'] = '1'
