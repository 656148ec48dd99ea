"""GW solve time on the BASELINE configs (the second half of the BASELINE metric).

    python tools/solve_bench.py c1            # full C1 solve through solve_cnt_gw
    python tools/solve_bench.py c4 [n] [outer] # C4 law, fixed 100-sweep inner budget
    python tools/solve_bench.py c5 [n] [outer] # C5 law, fixed 200-sweep inner budget
    python tools/solve_bench.py c3 [n]         # C3 eps-stage loop (tau = 1e-5)
    python tools/solve_bench.py ms [n]         # multiscale vs direct, C1 law

C4/C5 time the fixed number of outer steps the config names, stepping the
solver state without the stop rule (the cold laws trip the reference's own
divergence guard before step 10); wall time with a device
synchronize at each end, inputs already resident. Prints one JSON line.
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P  # noqa: E402
from paper_2602_06658_b200 import configs, solvers  # noqa: E402


def measures(pc):
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=pc.x.shape[1])
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=pc.y.shape[1])
    return src, tgt


def timed_steps(src, tgt, cfg, steps):
    st = solvers._CntGwState(src, tgt, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    objs, iters = [], []
    global STEP_S
    STEP_S = []
    for _ in range(steps):
        t1 = time.perf_counter()
        s = st.step()  # (ends with a host read of the reductions: synchronised)
        STEP_S.append(round(time.perf_counter() - t1, 3))
        objs.append(s.objective)
        iters.append(s.inner_iters)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, objs, iters, st.dev.prec


def main():
    which = sys.argv[1]
    args = [int(a) for a in sys.argv[2:]]
    torch.cuda.set_device(0)
    if which == "c1":
        pc = configs.c1(seed=0)
        src, tgt = measures(pc)
        cfg = P.make_config(configs.C1_EPS, threshold=1e-5, max_inner=200, max_outer=20)
        P.solve_cnt_gw(src, tgt, cfg)  # warm-up (graph capture, allocations)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = P.solve_cnt_gw(src, tgt, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out = dict(config="C1", n=1000, seconds=dt, outer=len(res.trace), value=res.value,
                   inner_iters=res.trace.inner_iters)
    elif which in ("c4", "c5"):
        n = args[0] if args else (1 << 20 if which == "c4" else 1 << 18)
        outer = args[1] if len(args) > 1 else 10
        pc = configs.GENERATORS[which.upper()](seed=0, n=n)
        src, tgt = measures(pc)
        eps, inner = (configs.C4_EPS, 100) if which == "c4" else (configs.C5_EPS, 200)
        cfg = P.make_config(eps, n_inner=inner, max_outer=outer)
        dt, objs, iters, prec = timed_steps(src, tgt, cfg, outer)
        passes = outer * (2 * inner + 2)
        out = dict(config=which.upper(), n=n, seconds=dt, outer=outer, inner=inner,
                   objectives=objs, precision_path=int(prec), step_seconds=STEP_S,
                   pairs_per_s=passes * float(n) * n / dt)
    elif which == "c3":
        n = args[0] if args else 100_000
        pc = configs.c3(seed=0, n=n)
        src, tgt = measures(pc)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prev, values, err = None, [], ""
        from dataclasses import replace

        for eps in configs.C3_EPS_STAGES:
            cfg = P.make_config(eps, threshold=1e-5, max_outer=10)
            warm = None
            if prev is not None:
                cfg = replace(cfg, init="gamma", init_gamma=prev.gamma)
                warm = (prev.coupling.f, prev.coupling.g)
            try:
                prev = P.solve_cnt_gw(src, tgt, cfg, _warm_potentials=warm)
            except P.SolverError as exc:
                err = f"{eps}: {exc}"
                break
            values.append(prev.value)
        torch.cuda.synchronize()
        out = dict(config="C3", n=n, seconds=time.perf_counter() - t0, stage_values=values,
                   error=err)
    elif which == "ms":
        # multiscale front end on the C1 law at larger N: k-means coarsening
        # (rho = 0.1) + coarse + fine solve, against the direct solve
        from paper_2602_06658_b200 import multiscale

        n = args[0] if args else 100_000
        pc = configs.c1(seed=0, n=n)
        src, tgt = measures(pc)
        cfg = P.make_config(configs.C1_EPS, threshold=1e-5, max_inner=200, max_outer=20)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rng = np.random.default_rng(cfg.seed)
        multiscale.coarsen(src, 0.1, rng)
        torch.cuda.synchronize()
        t_km = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = P.solve_multiscale(src, tgt, cfg, rho=0.1)
        torch.cuda.synchronize()
        t_ms = time.perf_counter() - t0
        t0 = time.perf_counter()
        direct = P.solve_cnt_gw(src, tgt, cfg)
        torch.cuda.synchronize()
        t_dir = time.perf_counter() - t0
        out = dict(config="C1-law multiscale", n=n, k=int(np.ceil(0.1 * n)),
                   kmeans_one_side_s=t_km, multiscale_s=t_ms, direct_s=t_dir,
                   multiscale_value=res.value, direct_value=direct.value,
                   fine_inner=res.trace.inner_iters, coarse_inner=res.coarse.trace.inner_iters,
                   direct_inner=direct.trace.inner_iters)
    else:
        raise SystemExit(f"unknown config {which}")
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
