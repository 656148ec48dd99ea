"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [names...]

It imports ``cntgw`` read-only from /root/reference and writes small ``.npz``
fixtures next to this file. Inputs come from the seeded generators in
``paper_2602_06658_b200/configs.py`` (float32-rounded, so both sides see the
same representable values); the inputs are stored in the fixture as well so
the tests never regenerate them.
"""

from __future__ import annotations

import os
import sys
import time
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import cntgw  # noqa: E402  (reference, read-only)
import importlib  # noqa: E402

ref_sk = importlib.import_module("cntgw.sinkhorn")
from cntgw.divergence import fourth_moment  # noqa: E402

from paper_2602_06658_b200 import configs  # noqa: E402


def _embed(points, weights, dim):
    m = cntgw.DiscreteMeasure(points, weights)
    return cntgw.embed_measure(m, cntgw.CostSpec("sq_euclidean"), dim=dim)


def _argmax(coupling):
    """argmax_j of the reconstructed plan (first max) and the top-2 log gap."""
    cost, f, g, eps = coupling.cost, coupling.f, coupling.g, coupling.eps_eff
    lb = np.log(coupling.target_weights) + g / eps
    n = cost.shape[0]
    idx = np.empty(n, dtype=np.int64)
    gap = np.empty(n)
    for i0 in range(0, n, 1024):
        i1 = min(i0 + 1024, n)
        s = lb[None, :] - cost.rows(i0, i1) / eps
        j = np.argmax(s, axis=1)
        idx[i0:i1] = j
        r = np.arange(i1 - i0)
        top = s[r, j].copy()
        s[r, j] = -np.inf
        gap[i0:i1] = top - s.max(axis=1)
    return idx, gap


def _solve_record(res, src, tgt, extra):
    cp = res.coupling
    idx, gap = _argmax(cp)
    tr = res.trace
    out = dict(
        gamma=res.gamma, f=cp.f, g=cp.g, zbar=cp.cost._z, xbar=cp.cost._x, eps_eff=cp.eps_eff,
        value=res.value, converged=res.converged,
        objective=np.array(tr.objectives), gamma_delta=np.array(tr.gamma_deltas),
        marginal_err=np.array(tr.marginal_errs), inner_iters=np.array(tr.inner_iters),
        argmax=idx, argmax_gap=gap,
        x_feat=src.features, y_feat=tgt.features, a=src.weights, b=tgt.weights,
    )
    out.update(extra)
    return out


def gen_c1():
    pc = configs.c1(seed=0)
    src = _embed(pc.x, pc.a, 3)
    tgt = _embed(pc.y, pc.b, 3)
    cfg = cntgw.make_config(configs.C1_EPS, threshold=1e-5, max_inner=200, max_outer=20)
    t0 = time.perf_counter()
    res = cntgw.solve_cnt_gw(src, tgt, cfg)
    wall = time.perf_counter() - t0
    const = cntgw.constant_value(src, tgt)
    return _solve_record(res, src, tgt, dict(x=pc.x, y=pc.y, constant=const, wall_s=wall,
                                             fm_x=fourth_moment(src), fm_y=fourth_moment(tgt)))


def gen_law(name, n, eps, inner_kw, max_outer):
    """Reduced-N same-law trajectory: ``max_outer`` reference steps, no stop rule.

    The cold C4/C5 laws trip the reference's divergence guard (solvers.py:604-609)
    before 10 steps, so the trajectory is recorded by stepping the reference's
    ``_CntGwState`` directly, and the outcome of the stock ``solve_cnt_gw`` (value
    or the step at which it raises ``SolverError``) is recorded beside it.
    """
    solvers = importlib.import_module("cntgw.solvers")
    pc = configs.GENERATORS[name](seed=0, n=n)
    dx, dy = pc.x.shape[1], pc.y.shape[1]
    src = _embed(pc.x, pc.a, dx)
    tgt = _embed(pc.y, pc.b, dy)
    cfg = cntgw.make_config(eps, max_outer=max_outer, **inner_kw)
    t0 = time.perf_counter()
    st = solvers._CntGwState(src, tgt, cfg)
    rec = {k: [] for k in ("objective", "gamma_delta", "marginal_err", "inner_iters",
                           "f_steps", "g_steps", "gamma_steps")}
    for _ in range(max_outer):
        s = st.step()
        rec["objective"].append(s.objective)
        rec["gamma_delta"].append(s.gamma_delta)
        rec["marginal_err"].append(s.marginal_err)
        rec["inner_iters"].append(s.inner_iters)
        rec["f_steps"].append(np.array(st.f))
        rec["g_steps"].append(np.array(st.g))
        rec["gamma_steps"].append(np.array(st.gamma))
    wall = time.perf_counter() - t0
    cp = st.coupling
    idx, gap = _argmax(cp)
    # stock outer-loop outcome on the same inputs
    try:
        res = cntgw.solve_cnt_gw(src, tgt, cfg)
        outcome, outcome_steps = "ok", len(res.trace)
    except cntgw.SolverError as exc:
        outcome, outcome_steps = f"SolverError: {exc}", -1
    # the step at which the guard fires, replayed from the recorded objectives
    ups, raise_at, prev = 0, -1, None
    for k, obj in enumerate(rec["objective"], start=1):
        if prev is not None:
            ch = prev - obj
            if abs(ch) < cfg.delta_outer:
                break
            ups = ups + 1 if ch < 0 else 0
            if ups >= 5:
                raise_at = k
                break
        prev = obj
    out = dict(
        gamma=st.gamma, f=cp.f, g=cp.g, zbar=cp.cost._z, xbar=cp.cost._x, eps_eff=cp.eps_eff,
        argmax=idx, argmax_gap=gap, x=pc.x, y=pc.y, x_feat=src.features, y_feat=tgt.features,
        a=src.weights, b=tgt.weights, constant=st.constant, wall_s=wall,
        fm_x=fourth_moment(src), fm_y=fourth_moment(tgt), outcome=np.array(outcome),
        outcome_steps=outcome_steps, raise_at=raise_at,
    )
    out.update({k: np.array(v) for k, v in rec.items()})
    return out


def gen_c3_stages(n=400, tau=1e-5, max_outer=10):
    """C3 eps-stage loop: warm potentials + init='gamma' per stage."""
    pc = configs.c3(seed=0, n=n)
    src = _embed(pc.x, pc.a, 3)
    tgt = _embed(pc.y, pc.b, 3)
    prev = None
    values, stages_done, gammas, iters = [], [], [], []
    err = ""
    for eps in configs.C3_EPS_STAGES:
        cfg = cntgw.make_config(eps, threshold=tau, max_outer=max_outer)
        warm = None
        if prev is not None:
            cfg = replace(cfg, init="gamma", init_gamma=prev.gamma)
            warm = (prev.coupling.f, prev.coupling.g)
        try:
            res = cntgw.solve_cnt_gw(src, tgt, cfg, _warm_potentials=warm)
        except cntgw.SolverError as exc:
            err = f"{eps}: {exc}"
            break
        prev = res
        values.append(res.value)
        stages_done.append(eps)
        gammas.append(res.gamma)
        iters.append(np.array(res.trace.inner_iters))
    out = dict(x=pc.x, y=pc.y, x_feat=src.features, y_feat=tgt.features, a=src.weights,
               b=tgt.weights, values=np.array(values), stages=np.array(stages_done),
               gammas=np.array(gammas), error=np.array(err),
               inner_iters=np.concatenate(iters) if iters else np.zeros(0, int),
               stage_lengths=np.array([len(i) for i in iters]))
    if prev is not None:
        idx, gap = _argmax(prev.coupling)
        out.update(f=prev.coupling.f, g=prev.coupling.g, zbar=prev.coupling.cost._z,
                   xbar=prev.coupling.cost._x, eps_eff=prev.coupling.eps_eff, argmax=idx,
                   argmax_gap=gap)
    return out


def gen_c1_api():
    """The building-block API on C1 (SURVEY.md §8b entry points): pi_step at
    the reference's converged Gamma, gamma_step / egw_objective on its plan,
    and every plan consumer (marginals, Err, KL, <C, pi>, EOT value) on that
    plan and on the solve's final coupling."""
    pc = configs.c1(seed=0)
    src = _embed(pc.x, pc.a, 3)
    tgt = _embed(pc.y, pc.b, 3)
    cfg = cntgw.make_config(configs.C1_EPS, threshold=1e-5, max_inner=200, max_outer=20)
    res = cntgw.solve_cnt_gw(src, tgt, cfg)
    gamma = res.gamma
    inner = cntgw.SinkhornConfig(eps=configs.C1_EPS, threshold=1e-5, max_inner=200)
    pr = cntgw.pi_step(gamma, src, tgt, configs.C1_EPS, inner)
    cp = pr.coupling
    gamma_next = cntgw.gamma_step(cp, src, tgt)
    out = dict(
        x_feat=src.features, y_feat=tgt.features, a=src.weights, b=tgt.weights, gamma=gamma,
        pi_f=cp.f, pi_g=cp.g, pi_iters=pr.iterations, pi_err=pr.marginal_err,
        pi_converged=pr.converged, pi_eps_eff=cp.eps_eff, pi_xbar=cp.cost._x, pi_zbar=cp.cost._z,
        gamma_next=gamma_next,
        obj=cntgw.egw_objective(gamma, cp, src, tgt, configs.C1_EPS),
        obj_next=cntgw.egw_objective(gamma_next, cp, src, tgt, configs.C1_EPS),
        pi_kl=cntgw.kl_divergence(cp), pi_me=cntgw.marginal_error(cp),
        pi_row=cp.row_marginal(), pi_col=cp.col_marginal(),
        pi_tc=cntgw.transport_cost(cp), pi_eot=cntgw.eot_primal_value(cp),
    )
    rc = res.coupling
    out.update(res_f=rc.f, res_g=rc.g, res_xbar=rc.cost._x, res_zbar=rc.cost._z,
               res_eps_eff=rc.eps_eff, res_kl=cntgw.kl_divergence(rc),
               res_me=cntgw.marginal_error(rc), res_tc=cntgw.transport_cost(rc),
               res_row=rc.row_marginal(), res_col=rc.col_marginal())
    return out


class _RowSubsetProvider:
    """Reference cost-provider protocol over selected rows of the C2 cost."""

    def __init__(self, u, v, ra, cb, rows):
        self.u, self.v, self.ra, self.cb, self.idx = u, v, ra, cb, rows

    @property
    def shape(self):
        return self.idx.size, self.v.shape[0]

    def rows(self, i0, i1):
        sel = self.idx[i0:i1]
        return self.ra[sel, None] + self.cb[None, :] - 2.0 * (self.u[sel] @ self.v.T)


def gen_c2_subsample(n=1 << 20, k=16, n_rows=64, seed=0):
    """C2 f-update on a row subsample at full M, via the reference ``_softmin``."""
    inst = configs.c2(seed=seed, n=n, k=k)
    rng = np.random.default_rng(1234)
    rows = np.sort(rng.choice(n, size=n_rows, replace=False))
    u = inst.u.astype(np.float64)
    v = inst.v.astype(np.float64)
    ra = inst.row_sep.astype(np.float64)
    cb = inst.col_sep.astype(np.float64)
    prov = _RowSubsetProvider(u, v, ra, cb, rows)
    f_rows = ref_sk._softmin(prov, inst.log_wb, inst.g.astype(np.float64), inst.eps)
    return dict(rows=rows, f_rows=f_rows, n=n, k=k, seed=seed)


def gen_c2_small(n=512, k=16, seed=3):
    """Whole C2 rep at small N through the public ``sinkhorn`` (standard, n_inner=1)."""
    inst = configs.c2(seed=seed, n=n, k=k)
    u = inst.u.astype(np.float64)
    v = inst.v.astype(np.float64)
    ra = inst.row_sep.astype(np.float64)
    cb = inst.col_sep.astype(np.float64)
    dense = ra[:, None] + cb[None, :] - 2.0 * (u @ v.T)
    w = np.full(n, 1.0 / n)
    cfg = cntgw.SinkhornConfig(eps=inst.eps, mode="standard", n_inner=1).with_warm_start(
        np.zeros(n), inst.g.astype(np.float64))
    res = cntgw.sinkhorn(w, w, ref_sk.DenseCost(dense), cfg)
    return dict(u=inst.u, v=inst.v, ra=inst.row_sep, cb=inst.col_sep, g0=inst.g,
                f=res.coupling.f, g=res.coupling.g, eps=inst.eps,
                marginal_err=res.marginal_err)


def _instance(n, m, seed, scale=1.0):
    # same construction as the reference test helper (test_sinkhorn.py:17-24)
    rng = np.random.default_rng(seed)
    a = rng.random(n) + 0.3
    a /= a.sum()
    b = rng.random(m) + 0.3
    b /= b.sum()
    c = rng.random((n, m)) * scale
    return a, b, c


def gen_sinkhorn_cases():
    """Dense and sq-Euclidean sinkhorn runs covering modes, budgets, annealing."""
    cases = [
        ("dense_sym_fixed", dict(n=9, m=7, seed=4), dict(eps=0.3, mode="symmetrized", n_inner=40)),
        ("dense_std_fixed", dict(n=9, m=7, seed=4), dict(eps=0.3, mode="standard", n_inner=40)),
        ("dense_sym_tau", dict(n=10, m=12, seed=5), dict(eps=0.2, threshold=1e-6, max_inner=5000)),
        ("dense_std_tau", dict(n=10, m=12, seed=5), dict(eps=0.2, mode="standard", threshold=1e-6,
                                                        max_inner=5000)),
        ("dense_anneal", dict(n=6, m=6, seed=11), dict(eps=0.05, n_inner=500, anneal_from=1.0)),
        ("dense_anneal_trunc", dict(n=6, m=6, seed=12), dict(eps=0.01, n_inner=4, anneal_from=1.0)),
        ("dense_cap", dict(n=8, m=8, seed=7), dict(eps=0.01, threshold=1e-14, max_inner=3)),
        ("dense_big", dict(n=300, m=257, seed=21), dict(eps=0.05, n_inner=30)),
    ]
    out = {}
    for name, inst, kw in cases:
        a, b, c = _instance(**inst)
        res = cntgw.sinkhorn(a, b, ref_sk.DenseCost(c), cntgw.SinkhornConfig(**kw))
        out[f"{name}__a"] = a
        out[f"{name}__b"] = b
        out[f"{name}__c"] = c
        out[f"{name}__f"] = res.coupling.f
        out[f"{name}__g"] = res.coupling.g
        out[f"{name}__iters"] = res.iterations
        out[f"{name}__conv"] = res.converged
        out[f"{name}__err"] = res.marginal_err
        out[f"{name}__eps_eff"] = res.coupling.eps_eff
        out[f"{name}__kw"] = repr(kw)
    # squared-Euclidean provider, symmetrized, both orientations
    rng = np.random.default_rng(9)
    x = rng.standard_normal((40, 3)).astype(np.float32).astype(np.float64)
    z = rng.standard_normal((33, 3)).astype(np.float32).astype(np.float64)
    a = np.full(40, 1.0 / 40)
    b = np.full(33, 1.0 / 33)
    res = cntgw.sinkhorn(a, b, ref_sk.SquaredEuclideanCost(x, z),
                         cntgw.SinkhornConfig(eps=0.4, mode="symmetrized", n_inner=21))
    out.update(sqe__x=x, sqe__z=z, sqe__f=res.coupling.f, sqe__g=res.coupling.g,
               sqe__err=res.marginal_err)
    return out


def gen_gradients():
    """Plan reductions, loss decomposition, envelope gradients, SGW and a short
    gradient flow (reference divergence.py:72-410) on C1-law clouds."""
    from cntgw import divergence as dv

    pc = configs.c1(seed=3, n=300, m=240)
    src = _embed(pc.x, pc.a, 3)
    tgt = _embed(pc.y, pc.b, 3)
    cfg = cntgw.make_config(0.05, n_inner=60, max_outer=6, delta_outer=1e-12)
    res = cntgw.solve_cnt_gw(src, tgt, cfg)
    pi_y, pi_sy, pit_x, pit_sx, sigma_ss = dv._plan_reductions(res.coupling, src, tgt)
    gsrc, gtgt = dv.feature_gradients(src, tgt, res.gamma, res.coupling)
    rep = dv.gw_value_report(res.gamma, res.coupling, src, tgt, 0.05)
    ql = dv.quartic_loss(res.coupling, src, tgt)
    gc = dv._grad_constant(src, tgt.trace_second_moment())
    sg = dv.sgw(src, tgt, cfg)
    rng = np.random.default_rng(11)
    pts = (rng.standard_normal((40, 3)) * 0.5).astype(np.float32).astype(np.float64)
    tpts = (rng.standard_normal((50, 3)) * 0.6).astype(np.float32).astype(np.float64)
    tau = _embed(tpts, np.full(50, 1.0 / 50), 3)
    fcfg = cntgw.make_config(0.1, n_inner=40, max_outer=4, delta_outer=1e-12)
    fl = dv.gradient_flow(cntgw.DiscreteMeasure(pts, np.full(40, 1.0 / 40)), [(1.0, tau)], fcfg,
                          steps=3, step_size=0.05)
    return dict(x_feat=src.features, y_feat=tgt.features, a=src.weights, b=tgt.weights,
                gamma=res.gamma, value=res.value, f=res.coupling.f, g=res.coupling.g,
                zbar=res.coupling.cost._z, eps_eff=res.coupling.eps_eff,
                pi_y=pi_y, pi_sy=pi_sy, pit_x=pit_x, pit_sx=pit_sx, sigma_ss=sigma_ss,
                gsrc=gsrc, gtgt=gtgt, grad_const=gc, quartic=ql,
                report=np.array([rep.value, rep.constant, rep.gamma_sq, rep.kl_term,
                                 rep.cross_term, rep.sigma_ss]),
                sgw_value=sg.value, sgw_parts=np.array([sg.cross.value, sg.self_src.value,
                                                        sg.self_tgt.value]),
                flow_points=pts, flow_tau=tpts, flow_positions=np.array(fl.positions),
                flow_objectives=np.array(fl.objectives))


def gen_multiscale():
    """Weighted k-means (incl. empty clusters and D=64), coarsen and the
    two-stage solve (reference solvers.py:668-763)."""
    from cntgw import solvers as rs

    out = {}
    rng = np.random.default_rng(21)
    cases = {}
    pc = configs.c1(seed=5, n=1000)
    cases["c1"] = (np.ascontiguousarray(pc.x - pc.x.mean(0)), np.full(1000, 1e-3), 100)
    xw = (rng.standard_normal((600, 3)) * [1.0, 0.5, 2.0]).astype(np.float32).astype(np.float64)
    ww = rng.dirichlet(np.ones(600))
    cases["dirichlet"] = (xw, ww, 37)
    base = (rng.standard_normal((3, 2))).astype(np.float32).astype(np.float64)
    xd = base[rng.integers(0, 3, 24)]
    cases["dupes"] = (xd, np.full(24, 1.0 / 24), 6)
    x64 = (rng.standard_normal((300, 64)) * 0.7).astype(np.float32).astype(np.float64)
    cases["d64"] = (x64, np.full(300, 1.0 / 300), 20)
    xb = (rng.standard_normal((3000, 3))).astype(np.float32).astype(np.float64)
    cases["bigclusters"] = (xb, rng.dirichlet(np.ones(3000)), 3)  # > 128 members: pairwise recursion
    for name, (x, w, k) in cases.items():
        assign, centers, cw = rs._weighted_kmeans(x, w, k, np.random.default_rng(7))
        out.update({f"{name}__x": x, f"{name}__w": w, f"{name}__k": np.array(k),
                    f"{name}__assign": assign, f"{name}__centers": centers, f"{name}__cw": cw})
    pc = configs.c1(seed=0)
    src = _embed(pc.x, pc.a, 3)
    tgt = _embed(pc.y, pc.b, 3)
    cfg = cntgw.make_config(configs.C1_EPS, threshold=1e-5, max_inner=200, max_outer=20)
    res = rs.solve_multiscale(src, tgt, cfg, rho=0.1)
    out.update(ms_x=src.features, ms_y=tgt.features, ms_a=src.weights, ms_b=tgt.weights,
               ms_value=res.value, ms_gamma=res.gamma, ms_f=res.coupling.f, ms_g=res.coupling.g,
               ms_inner=np.array(res.trace.inner_iters), ms_coarse_value=res.coarse.value,
               ms_coarse_gamma=res.coarse.gamma, ms_coarse_inner=np.array(res.coarse.trace.inner_iters))
    return out


def gen_kpca():
    """Kernel-PCA embeddings for every cost kind (dense branch, N=300), the
    subspace branch (N=4500 > 4096), centred kernels, the CNT diagnostic, cost
    matrices and gradients (reference kernels.py:149-446)."""
    from cntgw import kernels as rk

    rng = np.random.default_rng(8)
    pts = (rng.standard_normal((300, 5)) * [1.0, 0.8, 0.6, 0.4, 0.2]).astype(np.float32).astype(np.float64)
    w = rng.dirichlet(np.ones(300))
    emb6 = (rng.standard_normal((300, 6))).astype(np.float32).astype(np.float64)
    meas = cntgw.DiscreteMeasure(pts, w)
    dense_c = rk.cost_matrix(rk.CostSpec("euclidean"), meas)
    specs = {
        "euclid": (rk.CostSpec("euclidean"), 4),
        "pnorm": (rk.CostSpec("p_norm", p=1.5), 4),
        "exp": (rk.CostSpec("exp_kernel", sigma=0.8), 4),
        "sqlow": (rk.CostSpec("sq_euclidean"), 2),
        "embed": (rk.CostSpec("precomputed_embedding", path="mem", payload=emb6), 3),
        "matrix": (rk.CostSpec("dense_matrix", path="mem", payload=dense_c), 4),
    }
    out = dict(pts=pts, w=w, emb6=emb6)  # the dense_matrix payload is the euclidean cost of pts
    for name, (spec, dim) in specs.items():
        e = rk.embed_measure(meas, spec, dim=dim)
        out.update({f"{name}__f": e.features, f"{name}__ev": np.array(e.explained_variance),
                    f"{name}__vals": e.eigenvalues, f"{name}__dim": np.array(dim)})
    big = (rng.standard_normal((4500, 3)) * [1.0, 0.7, 0.4]).astype(np.float32).astype(np.float64)
    wb = np.full(4500, 1.0 / 4500)
    eb = rk.embed_measure(cntgw.DiscreteMeasure(big, wb), rk.CostSpec("euclidean"), dim=3)
    out.update(big=big, big__f=eb.features, big__vals=eb.eigenvalues, big__ev=np.array(eb.explained_variance))
    small = pts[:40]
    ws = np.full(40, 1.0 / 40)
    c40 = rk.cost_matrix(rk.CostSpec("euclidean"), cntgw.DiscreteMeasure(small, ws))
    kern = rk.kernel_from_cost(c40, ws, base_index=3)
    diag = rk.cnt_diagnostic(c40, ws)
    rnd = rng.random((40, 40))
    rnd = rnd + rnd.T
    np.fill_diagonal(rnd, 0.0)
    diag2 = rk.cnt_diagnostic(rnd, ws)
    out.update(c40=c40, k40=kern.matrix, diag=np.array([diag.min_eigenvalue, diag.max_abs_eigenvalue,
                                                         float(diag.is_cnt)]),
               rnd=rnd, diag2=np.array([diag2.min_eigenvalue, diag2.max_abs_eigenvalue, float(diag2.is_cnt)]),
               cexp=rk.cost_matrix(rk.CostSpec("exp_kernel", sigma=0.8), cntgw.DiscreteMeasure(small, ws)),
               gexp=rk.cost_gradients(rk.CostSpec("exp_kernel", sigma=0.8), small[:20]),
               gpn=rk.cost_gradients(rk.CostSpec("p_norm", p=1.5), small[:20]))
    return out


def gen_dense():
    """Dense-plan baselines: kernel-trick EGW and classical Entropic-GW, plus the
    adaptive wrapper around the kernel solver (reference solvers.py:384-665)."""
    from cntgw import kernels as rk
    from cntgw import solvers as rs

    pc = configs.c1(seed=9, n=120, m=100)
    mx = cntgw.DiscreteMeasure(pc.x, pc.a)
    my = cntgw.DiscreteMeasure(pc.y, pc.b)
    cx = rk.cost_matrix(rk.CostSpec("sq_euclidean"), mx)
    cy = rk.cost_matrix(rk.CostSpec("euclidean"), my)
    cfg = cntgw.make_config(0.05, n_inner=40, max_outer=6, delta_outer=1e-12)
    out = dict(x=pc.x, y=pc.y, a=pc.a, b=pc.b)
    for name, fn in (("kgw", rs.solve_kernel_gw), ("egw", rs.solve_entropic_gw)):
        res = fn(cx, cy, pc.a, pc.b, cfg)
        out.update({f"{name}__value": res.value, f"{name}__obj": np.array(res.trace.objectives),
                    f"{name}__delta": np.array(res.trace.gamma_deltas),
                    f"{name}__err": np.array(res.trace.marginal_errs),
                    f"{name}__pi": res.coupling.matrix})
    acfg = cntgw.make_config(0.05, n_inner=3, max_outer=8, delta_outer=1e-12)
    ares = rs.solve_adaptive(rs.solve_kernel_gw, cx, cy, pc.a, pc.b, cfg=acfg)
    out.update(ad__obj=np.array(ares.trace.objectives), ad__sched=np.array(ares.schedule))
    return out


GENS = {
    "c1_solve": gen_c1,
    "c4law_solve": lambda: gen_law("C4", 1024, configs.C4_EPS, dict(n_inner=100), 10),
    "c5law_solve": lambda: gen_law("C5", 256, configs.C5_EPS, dict(n_inner=200), 10),
    "c3law_stages": gen_c3_stages,
    "c1_api": gen_c1_api,
    "c2_subsample": gen_c2_subsample,
    "c2_small": gen_c2_small,
    "sinkhorn_cases": gen_sinkhorn_cases,
    "gradients": gen_gradients,
    "multiscale": gen_multiscale,
    "kpca": gen_kpca,
    "dense": gen_dense,
}


def main(names):
    for name in names or list(GENS):
        t0 = time.perf_counter()
        data = GENS[name]()
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
        print(f"{name}: {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
