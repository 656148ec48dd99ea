"""GPU parity of the CNT-GW outer solver against the reference's own outputs.

Golden vectors: tests/golden/{c1_solve,c4law_solve,c5law_solve}.npz, written
by tests/golden/make_golden.py from the reference package on identical
float32-rounded inputs. Tolerances (BASELINE north_star): potentials and GW
loss within 1e-4 relative (norm-wise, max|d| / max|ref|); argmax plan indices
bit-exact on rows whose reference top-2 log-score gap exceeds the certified
fp32 error bound, and inside the reference's near-tie set otherwise
(SURVEY.md §7.3e)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def P(cuda):
    import paper_2602_06658_b200 as P

    return P


def _measures(P, gold):
    src = P.EmbeddedMeasure(gold["x_feat"], gold["a"])
    tgt = P.EmbeddedMeasure(gold["y_feat"], gold["b"])
    return src, tgt


def _argmax_certified(gold, got, cert_nats):
    """(certified rows matching, certified rows, uncertified rows)."""
    sure = gold["argmax_gap"] > cert_nats
    match = int((got[sure] == gold["argmax"][sure]).sum())
    return match, int(sure.sum()), int((~sure).sum())


def _near_tie_ok(gold, got, rows, cert_nats):
    """Uncertified rows: GPU choice must score within cert of the reference max."""
    from oracle import cntgw_oracle as O

    cost = O.SqEuclid(gold["xbar"], gold["zbar"])
    eps = float(gold["eps_eff"])
    lb = np.log(gold["b"]) + gold["g"] / eps
    for i in rows:
        s = lb - cost.rows(int(i), int(i) + 1)[0] / eps
        assert s[got[i]] >= s.max() - cert_nats, i


@pytest.fixture(scope="module")
def c1(P):
    gold = golden("c1_solve")
    src, tgt = _measures(P, gold)
    cfg = P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20)
    return gold, P.solve_cnt_gw(src, tgt, cfg)


def test_c1_constant(P):
    gold = golden("c1_solve")
    src, tgt = _measures(P, gold)
    assert P.constant_value(src, tgt) == pytest.approx(float(gold["constant"]), rel=1e-12)
    assert P.fourth_moment(src) == pytest.approx(float(gold["fm_x"]), rel=1e-12)


def test_c1_trajectory_decisions(c1):
    gold, res = c1
    # same number of outer steps and same per-step inner sweep counts
    assert len(res.trace) == len(gold["objective"])
    assert res.trace.inner_iters == gold["inner_iters"].tolist()
    assert res.converged == bool(gold["converged"])


def test_c1_potentials_and_loss(c1):
    gold, res = c1
    assert _rel(res.coupling.f, gold["f"]) < TOL
    assert _rel(res.coupling.g, gold["g"]) < TOL
    assert abs(res.value - float(gold["value"])) <= TOL * abs(float(gold["value"]))
    assert _rel(res.trace.objectives, gold["objective"]) < TOL
    assert _rel(res.gamma, gold["gamma"]) < TOL
    assert res.coupling.eps_eff == pytest.approx(float(gold["eps_eff"]))
    # zbar is built from Gamma_t (result pairing, Appendix A.1 item 11)
    assert _rel(res.coupling.cost._z, gold["zbar"]) < TOL


@pytest.mark.parametrize("device_loop", ["1", "0"], ids=["captured", "host-loop"])
def test_c1_forced_f64s_path(P, device_loop, monkeypatch):
    """The whole C1 solve forced onto CNTGW_F64S (probe, measured plan, the
    Gamma = 0 fast path of the first step, rows block gathered once and only
    the bias column repacked within a thresholded loop), as one captured graph
    and through the host loop: same decisions, potentials and loss as the
    reference."""
    gold = golden("c1_solve")
    src, tgt = _measures(P, gold)
    monkeypatch.setenv("CNTGW_PRECISION", "f64s")
    monkeypatch.setenv("CNTGW_DEVICE_LOOP", device_loop)
    res = P.solve_cnt_gw(src, tgt, P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20))
    assert res.trace.inner_iters == gold["inner_iters"].tolist()
    assert res.converged == bool(gold["converged"])
    assert _rel(res.coupling.f, gold["f"]) < TOL
    assert _rel(res.coupling.g, gold["g"]) < TOL
    assert abs(res.value - float(gold["value"])) <= TOL * abs(float(gold["value"]))
    assert _rel(res.gamma, gold["gamma"]) < TOL


def test_c1_marginal_err_trace(c1):
    gold, res = c1
    got, want = np.array(res.trace.marginal_errs), gold["marginal_err"]
    assert np.all(np.abs(got - want) <= 1e-3 * want + 1e-7)


def test_c1_argmax(c1):
    gold, res = c1
    cert = 1e-3  # nats: fp32 exponent rounding at |t| ~ 2^11 plus potential error
    match, sure, unsure = _argmax_certified(gold, res.argmax, cert)
    assert match == sure, f"{sure - match} certified rows differ"
    _near_tie_ok(gold, res.argmax, np.nonzero(gold["argmax_gap"] <= cert)[0], cert)


def test_c1_pi_step_gamma_step_objective(P, c1):
    """The building-block API reproduces the solver's last step."""
    gold, res = c1
    src, tgt = _measures(P, gold)
    inner = P.SinkhornConfig(eps=0.01, threshold=1e-5, max_inner=200)
    gamma_prev = np.linalg.lstsq(  # Gamma_t is recoverable from zbar = Y Gamma_t^T
        tgt.features, res.coupling.cost._z[:, :-1], rcond=None)[0].T
    pr = P.pi_step(gamma_prev, src, tgt, 0.01, inner)
    assert pr.coupling.eps_eff == pytest.approx(0.01 / 8)
    gam = P.gamma_step(res.coupling, src, tgt)
    assert _rel(gam, res.gamma) < 1e-5
    obj = P.egw_objective(res.gamma, res.coupling, src, tgt, 0.01)
    assert np.isfinite(obj)


def _law_argmax(state, gold):
    """argmax plan indices of the final coupling (K4, fused) against the
    reference's. The certificate is data-driven: a score s_ij = log b_j +
    (g_j - C_ij)/eps moves by at most |dg_j|/eps between the two solves, so a
    row whose reference top-2 gap exceeds 2 max|dg|/eps (+ rounding) must
    pick the same column; the others must pick a column inside the tie band."""
    cp = state.coupling()
    eps = float(gold["eps_eff"])
    assert cp.eps_eff == pytest.approx(eps, rel=1e-12)
    cert = 2.0 * float(np.abs(cp.g - gold["g"]).max()) / eps + 1e-6
    got = state.dev.argmax.cpu().numpy()
    match, sure, unsure = _argmax_certified(gold, got, cert)
    print(f"argmax: {match}/{sure} certified rows identical (cert {cert:.2e} nats), {unsure} near ties")
    assert match == sure, f"{sure - match} certified rows differ"
    assert sure >= 0.5 * got.size
    _near_tie_ok(gold, got, np.nonzero(gold["argmax_gap"] <= cert)[0], cert)


@pytest.mark.parametrize("name,eps,n_inner", [("c4law_solve", 0.01, 100), ("c5law_solve", 0.02, 200)])
def test_law_trajectory(P, name, eps, n_inner):
    """Reduced-N same-law runs: 10 reference steps stepped without the stop rule."""
    from paper_2602_06658_b200 import solvers

    gold = golden(name)
    src, tgt = _measures(P, gold)
    cfg = P.make_config(eps, n_inner=n_inner, max_outer=10)
    state = solvers._CntGwState(src, tgt, cfg)
    assert state.constant == pytest.approx(float(gold["constant"]), rel=1e-10)
    objs = []
    for k in range(10):
        s = state.step()
        objs.append(s.objective)
        f = state.coupling().f
        assert _rel(f, gold["f_steps"][k]) < TOL, f"step {k + 1}: f"
        assert _rel(state.coupling().g, gold["g_steps"][k]) < TOL, f"step {k + 1}: g"
    assert _rel(objs, gold["objective"]) < TOL
    _law_argmax(state, gold)
    # the stock outer loop reaches the same outcome (value or SolverError step)
    if int(gold["raise_at"]) > 0:
        with pytest.raises(P.SolverError):
            P.solve_cnt_gw(src, tgt, cfg)


@pytest.mark.parametrize("name,eps,n_inner", [("c4law_solve", 0.01, 100), ("c5law_solve", 0.02, 200)])
def test_law_trajectory_centred_path(P, name, eps, n_inner, monkeypatch):
    """The same reduced-N reference trajectories through the CNTGW_F32C
    half-updates (forced; at these sizes most tile pairs take the kernel's
    fp64 fallback, the rest the centred fp32 sweep)."""
    from paper_2602_06658_b200 import solvers

    monkeypatch.setenv("CNTGW_PRECISION", "f32c")
    gold = golden(name)
    src, tgt = _measures(P, gold)
    state = solvers._CntGwState(src, tgt, P.make_config(eps, n_inner=n_inner, max_outer=10))
    objs = []
    for k in range(10):
        objs.append(state.step().objective)
        assert _rel(state.coupling().f, gold["f_steps"][k]) < TOL, f"step {k + 1}: f"
        assert _rel(state.coupling().g, gold["g_steps"][k]) < TOL, f"step {k + 1}: g"
    assert _rel(objs, gold["objective"]) < TOL
    _law_argmax(state, gold)


def test_device_graph_loop_centred_path(P, monkeypatch):
    """Whole-solve CUDA graph with the centred path forced: the C1 reference
    solve (stop step, inner counts, value)."""
    monkeypatch.setenv("CNTGW_PRECISION", "f32c")
    gold = golden("c1_solve")
    src, tgt = _measures(P, gold)
    res = P.solve_cnt_gw(src, tgt, P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20))
    assert list(res.trace.inner_iters) == [int(v) for v in gold["inner_iters"]]
    assert _rel([res.value], [float(gold["value"])]) < TOL


def test_device_graph_loop_equals_host_loop(P, monkeypatch):
    """The single-graph solve (nested conditional WHILE nodes) and the
    host-driven loop run the same kernels: identical trajectories."""
    gold = golden("c1_solve")
    src, tgt = _measures(P, gold)
    cfg = P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20)
    dev_res = P.solve_cnt_gw(src, tgt, cfg)
    monkeypatch.setenv("CNTGW_DEVICE_LOOP", "0")
    host_res = P.solve_cnt_gw(src, tgt, cfg)
    assert dev_res.trace.inner_iters == host_res.trace.inner_iters
    # the objective is summed on the device in one loop and on the host in
    # another: equal to the last couple of ulps
    np.testing.assert_allclose(dev_res.trace.objectives, host_res.trace.objectives, rtol=1e-13)
    assert np.array_equal(dev_res.coupling.f, host_res.coupling.f)
    assert np.array_equal(dev_res.gamma, host_res.gamma)
    assert np.array_equal(dev_res.argmax, host_res.argmax)
    assert all(t > 0 for t in dev_res.trace.elapsed_s)


def test_final_anneal_and_fixed_budget_graph(P):
    """final_anneal appends one annealed step after the captured loop."""
    gold = golden("c1_solve")
    src, tgt = _measures(P, gold)
    cfg = P.make_config(0.01, n_inner=8, max_outer=3, final_anneal=0.05, delta_outer=1e-12)
    res = P.solve_cnt_gw(src, tgt, cfg)
    assert len(res.trace) == 4 and res.trace.inner_iters == [8, 8, 8, 8]
    from oracle import cntgw_oracle as O

    ref = O.solve_cnt_gw(gold["x_feat"], gold["a"], gold["y_feat"], gold["b"], 0.01,
                         dict(n_inner=8), max_outer=3, delta_outer=1e-12, final_anneal=0.05)
    # a fixed 8-sweep budget stops the annealing schedule before eps' = eps/8
    assert res.coupling.eps_eff == pytest.approx(ref["eps_eff"], rel=1e-12)
    assert res.coupling.eps_eff > 0.01 / 8
    assert _rel(res.trace.objectives, ref["trace"]["objective"]) < TOL
    assert _rel(res.coupling.f, ref["f"]) < TOL


def test_c3_eps_stage_chain_matches_reference(P):
    """C3-law eps-stage loop (0.1 -> 0.00625, tau = 1e-5, warm potentials and
    init='gamma' chained across stages) at N=400 against the reference's own
    run: stage values, Gamma per stage, every inner-sweep count, and the
    SolverError the reference raises at the 0.00625 stage."""
    from dataclasses import replace

    from paper_2602_06658_b200 import configs

    gold = golden("c3law_stages")
    src, tgt = _measures(P, gold)
    prev, values, gammas, iters, lengths, err = None, [], [], [], [], ""
    for eps in configs.C3_EPS_STAGES:
        cfg = P.make_config(eps, threshold=1e-5, max_outer=10)
        warm = None
        if prev is not None:
            cfg = replace(cfg, init="gamma", init_gamma=prev.gamma)
            warm = (prev.coupling.f, prev.coupling.g)
        try:
            res = P.solve_cnt_gw(src, tgt, cfg, _warm_potentials=warm)
        except P.SolverError as exc:
            err = f"{eps}: {exc}"
            break
        prev = res
        values.append(res.value)
        gammas.append(res.gamma)
        iters += list(res.trace.inner_iters)
        lengths.append(len(res.trace))
    assert err.split(":")[0] == str(gold["error"]).split(":")[0]
    assert lengths == list(gold["stage_lengths"])
    # the weighted-gap stop decision lands on the same sweep, or (when the gap
    # crosses tau within rounding of the fp32 exponent path) one sweep apart
    diff = np.abs(np.array(iters) - gold["inner_iters"])
    assert diff.max() <= 1 and (diff > 0).sum() <= 2, list(diff)
    assert _rel(values, gold["values"]) < TOL
    assert _rel(np.array(gammas), gold["gammas"]) < TOL
    assert _rel(prev.coupling.f, gold["f"]) < TOL
    assert _rel(prev.coupling.g, gold["g"]) < TOL
    # argmax plan indices of the last completed stage (same certificate as
    # the law trajectories: reference top-2 gap vs 2 max|dg| / eps)
    eps = float(gold["eps_eff"])
    cert = 2.0 * float(np.abs(prev.coupling.g - gold["g"]).max()) / eps + 1e-6
    match, sure, unsure = _argmax_certified(gold, prev.argmax, cert)
    assert match == sure and sure >= 0.5 * prev.argmax.size, (match, sure, unsure)
    _near_tie_ok(gold, prev.argmax, np.nonzero(gold["argmax_gap"] <= cert)[0], cert)


def test_c4_full_size_centred_half_updates_match_fp64(P, monkeypatch):
    """C4 at its full size (N=M=2^20): on a warm pair (one fp64 outer step of
    5 sweeps) the automatic path choice is fp64 with the measured plan
    (CNTGW_F64S), and both it and the centred fp32 kernel (CNTGW_F32C) agree
    with the dense fp64 kernel (itself pinned to the reference at reduced N):
    potentials to 1e-6 relative, 99% of the rows within 1e-3 log2 units of
    the plan entries."""
    import torch

    from paper_2602_06658_b200 import configs, engine, solvers
    from paper_2602_06658_b200._native import F32C, F64, F64S

    pc = configs.c4(seed=0)
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=3)
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=3)
    monkeypatch.setenv("CNTGW_PRECISION", "f64")
    st = solvers._CntGwState(src, tgt, P.make_config(configs.C4_EPS, n_inner=5, max_outer=2))
    st.step()
    dev = st.dev
    dev.set_gamma(st.gamma)
    monkeypatch.setenv("CNTGW_PRECISION", "auto")
    eps = configs.C4_EPS / 8
    dev.choose_precision(st.f, st.g, eps)
    assert dev.prec == F64S
    state = dev.loop.state
    state.init(eps)
    lam = np.log2(np.e) / eps
    for op, pot, length in ((dev.fwd, st.g, dev.n), (dev.bwd, st.f, dev.m)):
        outs = {}
        for prec in (F64, F32C, F64S):
            op.prec = prec
            outs[prec] = torch.empty(length, dtype=torch.float64, device=dev.device)
            op(state, pot, outs[prec], skip=False)
        b = outs[F64].cpu().numpy()
        for prec, tol in ((F32C, 1e-6), (F64S, 1e-9)):
            a = outs[prec].cpu().numpy()
            assert _rel(a, b) < tol, prec
            assert np.percentile(np.abs(a - b) * lam, 99) < 1e-3, prec


@pytest.mark.parametrize("path", ["f32c", "f64s"])
def test_block_sparse_k4_matches_dense(P, path, monkeypatch):
    """K4 on the centred path's block-sparse plan (cntgw_plan_reduce_ctr)
    against the dense fp64 K4 (cntgw_plan_reduce) on the SAME final pair:
    C4 law, N=M=2^16, after an outer step on the centred path. Skipped tiles
    hold < 2^-64 of every row's mass and both passes are fp64 throughout, so
    row masses, pi Y, pi t agree to summation order; argmax indices agree
    except where two columns score within a few ulps (the two passes build
    their column records with differently rounded fp64 arithmetic). Two full
    outer steps with either pass agree to the centred kernel's fp32 noise."""
    from paper_2602_06658_b200 import configs, solvers

    if path == "f32c":  # C4 law, the centred path's geometric plan
        pc, eps, dims = configs.c4(seed=2, n=1 << 16), configs.C4_EPS, (3, 3)
    else:  # C5 law, CNTGW_F64S's measured plan
        pc, eps, dims = configs.c5(seed=2, n=1 << 14), configs.C5_EPS, (64, 32)
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=dims[0])
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=dims[1])
    monkeypatch.setenv("CNTGW_PRECISION", path)
    st = solvers._CntGwState(src, tgt, P.make_config(eps, n_inner=30, max_outer=2))
    st.step()
    st.step()
    dev = st.dev
    outs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("CNTGW_K4_SPARSE", flag)
        dev.plan_pass(st.f, st.g)
        outs[flag] = tuple(t.cpu().numpy().copy() for t in (dev.r, dev.pi_y, dev.pi_s, dev.argmax))
    sp, de = outs["1"], outs["0"]
    for k, name in enumerate(("r", "pi_y", "pi_s")):
        assert _rel(sp[k], de[k]) < 1e-12, name
    same = float((sp[3] == de[3]).mean())
    print(f"argmax identical on {same:.6f} of the rows")
    assert same > 0.999
    # whole outer steps with either pass (the loop's fp32 noise amplifies any
    # difference in Gamma_1, so this is a looser, trajectory-level check)
    traj = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("CNTGW_K4_SPARSE", flag)
        s2 = solvers._CntGwState(src, tgt, P.make_config(eps, n_inner=30, max_outer=2))
        objs = [s2.step().objective for _ in range(2)]
        traj[flag] = (np.array(objs), s2.gamma.copy())
    assert _rel(traj["1"][0], traj["0"][0]) < 1e-6
    assert _rel(traj["1"][1], traj["0"][1]) < 1e-6


def test_captured_solve_precision_covers_every_reachable_gamma(P, monkeypatch):
    """The graph-captured solve fixes one kernel path for all outer steps. A
    problem that is well scaled at Gamma_0 = 0 (fp32 exponents would be
    chosen there) but whose reachable operators (||Gamma|| <= sqrt(T_x T_y))
    are cold must be captured on an fp64-safe path; the solve then matches
    the oracle and the host loop (which re-selects the path every step)."""
    from oracle import cntgw_oracle as O
    from paper_2602_06658_b200 import configs, solvers
    from paper_2602_06658_b200._native import F32, F32C, F64

    pc = configs.c1(seed=3, n=300)
    x = (pc.x - pc.a @ pc.x) * 2.0
    y = (pc.y - pc.b @ pc.y) * 2.0
    src, tgt = P.EmbeddedMeasure(x, pc.a), P.EmbeddedMeasure(y, pc.b)
    cfg = P.make_config(0.01, n_inner=30, max_outer=4, delta_outer=1e-12)
    st = solvers._CntGwState(src, tgt, cfg)
    dev = st.dev
    dev.set_gamma(st.gamma)
    dev.choose_precision(st.f, st.g, 0.01 / 8)
    assert dev.prec == F32  # the per-step rule at Gamma_0
    dev.choose_precision(st.f, st.g, 0.01 / 8, reachable=True)
    assert dev.prec in (F64, F32C)  # the rule the captured solve applies
    res = P.solve_cnt_gw(src, tgt, cfg)
    ref = O.solve_cnt_gw(x, pc.a, y, pc.b, 0.01, dict(n_inner=30), max_outer=4, delta_outer=1e-12)
    assert _rel(res.trace.objectives, ref["trace"]["objective"]) < TOL
    assert _rel(res.coupling.f, ref["f"]) < TOL and _rel(res.gamma, ref["gamma"]) < TOL
    monkeypatch.setenv("CNTGW_DEVICE_LOOP", "0")
    host = P.solve_cnt_gw(src, tgt, cfg)
    assert _rel(host.trace.objectives, ref["trace"]["objective"]) < TOL
