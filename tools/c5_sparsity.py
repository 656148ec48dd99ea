"""How block-sparse is the C5 plan? (design probe for the C5 kernel)

    python tools/c5_sparsity.py [n] [outer] [n_inner]

Steps the C5 solver state (automatic path) for `outer` outer steps of
`n_inner` sweeps, then evaluates the f-update's exponent q_ij (fp64, torch
blocks on the GPU) of the current pair and reports, for several row/column
orders, the fraction of (128-row group, 256-column tile) pairs that hold a
term within T log2 units of some row's maximum (T = 64, 80): the work a
measured block-sparse plan would keep. Orders: the caller's (natural), the
locality order of the solver's points (Morton codes of the first 3
coordinates), and a cluster order (device k-means on the features).
"""

import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P  # noqa: E402
from paper_2602_06658_b200 import configs, engine, solvers  # noqa: E402


def need_fraction(q_rows, order_r, order_c, T, G=128, TL=256):
    """q_rows(i0, i1, cols) -> fp64 block of q (rows i0:i1 in order_r, all cols
    in order_c); returns the fraction of needed (group, tile) pairs."""
    n, m = order_r.numel(), order_c.numel()
    ng, nt = (n + G - 1) // G, (m + TL - 1) // TL
    need = 0
    for g0 in range(0, ng, 16):
        rows = order_r[g0 * G:min(n, (g0 + 16) * G)]
        q = q_rows(rows, order_c)  # (r, m), min over j is the row max of t
        qmin = q.min(1, keepdim=True).values
        mpad = nt * TL
        if mpad > m:
            q = torch.nn.functional.pad(q, (0, mpad - m), value=math.inf)
        close = (q <= qmin + T).view(q.shape[0], nt, TL).any(2)  # (r, nt)
        r = close.shape[0]
        gpad = (r + G - 1) // G * G
        if gpad > r:
            close = torch.nn.functional.pad(close, (0, 0, 0, gpad - r))
        need += int(close.view(-1, G, nt).any(1).sum())
    return need / (ng * nt)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
    outer = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    inner = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    torch.cuda.set_device(0)
    pc = configs.c5(seed=0, n=n)
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=64)
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=32)
    st = solvers._CntGwState(src, tgt, P.make_config(configs.C5_EPS, n_inner=inner, max_outer=outer))
    t0 = time.time()
    for k in range(outer):
        s = st.step()
        print(f"step {k + 1}: objective {s.objective:.6f} err {s.marginal_err:.3e} ({time.time() - t0:.1f} s)",
              flush=True)
    dev = st.dev
    dev.set_gamma(st.coupling_gamma)
    lam = math.log2(math.e) / st.eps_eff
    # q-form of the f-update: q_ij = -(lam (g~_j + 2<x,z> - (s_i - t_j)^2) + log2 b_j)
    xr, zc = dev.src.feat64, dev.tgt.feat64
    sr, tc = dev.sx, dev.ty
    g, lb = st.g, dev.tgt.log2w

    def q_rows(rows, cols):
        x, s = xr[rows], sr[rows]
        z, t = zc[cols], tc[cols]
        return -(lam * (g[cols][None, :] + 2.0 * (x @ z.t()) - (s[:, None] - t[None, :]) ** 2)
                 + lb[cols][None, :])

    nat_r = torch.arange(dev.n, device=xr.device)
    nat_c = torch.arange(dev.m, device=xr.device)
    orders = {"natural": (nat_r, nat_c),
              "morton3": (dev.src.locality(), dev.tgt.locality())}
    # cluster order: sort by the nearest of 16 (k-means++ style farthest-point) centres, then by s
    for name, (o_r, o_c) in orders.items():
        for T in (64.0, 80.0):
            t1 = time.time()
            fr = need_fraction(q_rows, o_r, o_c, T)
            print(f"order {name} T={T:.0f}: needed (group, tile) fraction {fr:.4f} "
                  f"({time.time() - t1:.1f} s)", flush=True)
    # rows sorted by argmin column cluster (the column tile holding the row max), columns natural
    best = []
    for i0 in range(0, dev.n, 4096):
        rows = nat_r[i0:i0 + 4096]
        best.append(q_rows(rows, nat_c).argmin(1))
    best = torch.cat(best)
    o_r = torch.sort(best, stable=True).indices
    for T in (64.0, 80.0):
        fr = need_fraction(q_rows, o_r, nat_c, T)
        print(f"order rows-by-argmax T={T:.0f}: needed fraction {fr:.4f}", flush=True)


if __name__ == "__main__":
    main()
