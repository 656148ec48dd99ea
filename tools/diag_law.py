"""Per-step parity diagnostics of the GPU solver against a reduced-N golden
trajectory: full-trajectory errors and one-step errors (each GPU step started
from the reference's own state). Usage: python tools/diag_law.py c4law_solve 0.01 100"""

import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2602_06658_b200 as P  # noqa: E402
from paper_2602_06658_b200 import engine, solvers  # noqa: E402


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def main(name, eps, n_inner, steps=10):
    g = dict(np.load(f"tests/golden/{name}.npz"))
    src, tgt = P.EmbeddedMeasure(g["x_feat"], g["a"]), P.EmbeddedMeasure(g["y_feat"], g["b"])
    cfg = P.make_config(eps, n_inner=n_inner, max_outer=steps)
    st = solvers._CntGwState(src, tgt, cfg)
    print(f"constant rel err {abs(st.constant - float(g['constant'])) / abs(float(g['constant'])):.2e}")
    print("full trajectory: step  f  g  gamma  objective")
    for k in range(steps):
        s = st.step()
        cp = st.coupling()
        print(f"  {k + 1:2d} {rel(cp.f, g['f_steps'][k]):.2e} {rel(cp.g, g['g_steps'][k]):.2e} "
              f"{rel(st.gamma, g['gamma_steps'][k]):.2e} "
              f"{abs(s.objective - g['objective'][k]) / abs(g['objective'][k]):.2e}")
    print("one-step (from the reference state): step  f  g  gamma  objective")
    dev = st.dev
    for k in range(steps):
        if k == 0:
            gamma_prev, gamma_cur = np.zeros_like(g["gamma_steps"][0]), np.zeros_like(g["gamma_steps"][0])
            st2 = solvers._CntGwState(src, tgt, cfg)
        else:
            gamma_cur = g["gamma_steps"][k - 1]
            gamma_prev = g["gamma_steps"][k - 2] if k >= 2 else np.zeros_like(gamma_cur)
            f_ref = engine.to_dev64(g["f_steps"][k - 1], dev.device)
            g_ref = engine.to_dev64(g["g_steps"][k - 1], dev.device)
            st2.gamma = gamma_cur
            st2.f.copy_(f_ref - st2.dev.row_sep())
            st2.g.copy_(g_ref - st2.dev.col_sep(gamma_prev))
        s = st2.step()
        cp = st2.coupling()
        print(f"  {k + 1:2d} {rel(cp.f, g['f_steps'][k]):.2e} {rel(cp.g, g['g_steps'][k]):.2e} "
              f"{rel(st2.gamma, g['gamma_steps'][k]):.2e} "
              f"{abs(s.objective - g['objective'][k]) / abs(g['objective'][k]):.2e}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]))
