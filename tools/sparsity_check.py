"""How many (row group, column tile) pairs of a centred half-update can be
skipped with a rigorous bound? (design probe for a block-sparse softmin)

    python tools/sparsity_check.py [n] [sweeps] [T]

On the C4 law after one outer step of `sweeps` sweeps: for every 128-row
group I and 256-column tile J (Morton order), rho_IJ = min_j A_j^I, the
pair-term bound C_IJ = R_I R_J, per row B_i^J; the row's max term is at least
L_i = max_J (-rho - B - C); tile J cannot hold a term above L_i - T for row i
when -rho - B + C < L_i - T. Prints the fraction of (group, tile) pairs, and
of (8-group CTA, tile) pairs, that hold no such term for any of their rows.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P  # noqa: E402
from paper_2602_06658_b200 import configs, engine, solvers  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    T = float(sys.argv[3]) if len(sys.argv) > 3 else 64.0
    torch.cuda.set_device(0)
    pc = configs.c4(seed=0, n=n)
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=3)
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=3)
    st = solvers._CntGwState(src, tgt, P.make_config(configs.C4_EPS, n_inner=sweeps, max_outer=2))
    st.step()
    dev = st.dev
    dev.set_gamma(st.gamma)
    eps = configs.C4_EPS / 8
    lam = np.log2(np.e) / eps
    out = {}
    for name, rows, cols, pot in (("f", dev.src, dev.tgt, st.g), ("g", dev.tgt, dev.src, st.f)):
        # fp64 features in locality order: X = [x | s], Zr = -2 lam [z | t], c
        X = torch.cat([rows.feat64, rows.sq64[:, None]], 1)[rows.locality()]
        Zf = torch.cat([cols.feat64, cols.sq64[:, None]], 1)[cols.locality()]
        t = cols.sq64[cols.locality()]
        c = -(lam * (pot[cols.locality()] - t * t) + cols.log2w[cols.locality()])
        Zr = -2.0 * lam * Zf
        nr, m = X.shape[0], Zr.shape[0]
        G, TL = nr // 128, m // 256
        X, Zr, c = X[: G * 128], Zr[: TL * 256], c[: TL * 256]
        Xg = X.view(G, 128, -1)
        Xc = Xg.mean(1)
        dX = Xg - Xc[:, None]
        RI = dX.norm(dim=2).amax(1)
        Zt = Zr.view(TL, 256, -1)
        Zc = Zt.mean(1)
        RJ = (Zt - Zc[:, None]).norm(dim=2).amax(1)
        rho = torch.empty(G, TL, dtype=torch.float64, device=X.device)
        for g0 in range(0, G, 64):
            A = c[None, :] + Xc[g0:g0 + 64] @ Zr.T
            rho[g0:g0 + 64] = A.view(-1, TL, 256).amin(2)
        C = RI[:, None] * RJ[None, :]
        # per row: L_i = max_J (-rho - B - C); keep_iJ = -rho - B + C >= L_i - T
        keep_g = torch.zeros(G, TL, dtype=torch.bool, device=X.device)
        for g0 in range(0, G, 32):
            B = torch.einsum("gik,jk->gij", dX[g0:g0 + 32], Zc)  # (32, 128, TL)
            base = -rho[g0:g0 + 32, None, :] - B
            L = (base - C[g0:g0 + 32, None, :]).amax(2, keepdim=True)
            keep = (base + C[g0:g0 + 32, None, :]) >= L - T
            keep_g[g0:g0 + 32] = keep.any(1)
        cta = keep_g[: G // 8 * 8].view(G // 8, 8, TL).any(1)
        out[name] = dict(group_tile_kept=float(keep_g.float().mean()), cta_tile_kept=float(cta.float().mean()))
    print(json.dumps(dict(n=n, sweeps=sweeps, T=T, kept=out)), flush=True)


if __name__ == "__main__":
    main()
