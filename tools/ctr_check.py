"""Centred fp32 path (CNTGW_F32C) against the fp64 path on a cold law.

    python tools/ctr_check.py [c4|c3|c5] [n] [outer] [inner]

Steps the CNT-GW state `outer` times with a fixed inner budget, once with
CNTGW_PRECISION=f64 and once with f32c, from the same inputs; prints per-step
relative differences of f, g, Gamma and the objective (norm-wise, as the
parity tests measure them), the wall time of each run, the pair-term bound
engine.centred_scale and the path the automatic choice takes. One JSON line.
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P  # noqa: E402
from paper_2602_06658_b200 import configs, engine, solvers  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def run(src, tgt, cfg, outer, prec):
    os.environ["CNTGW_PRECISION"] = prec
    st = solvers._CntGwState(src, tgt, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = []
    for _ in range(outer):
        s = st.step()
        c = st.coupling()
        out.append((s.objective, c.f.copy(), c.g.copy(), np.array(st.gamma, copy=True)))
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out, st


def half_update_error(which, n, warm_sweeps):
    """One f-update and one g-update with every path on the same warm pair:
    errors against the fp64 path in log2 units (lam * |delta|)."""
    from paper_2602_06658_b200._native import F32, F32C, F64
    eps = {"c4": configs.C4_EPS, "c5": configs.C5_EPS, "c3": configs.C3_EPS_STAGES[-1]}[which]
    pc = configs.GENERATORS[which.upper()](seed=0, n=n)
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=pc.x.shape[1])
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=pc.y.shape[1])
    os.environ["CNTGW_PRECISION"] = "f64"
    cfg = P.make_config(eps, n_inner=warm_sweeps, max_outer=2)
    st = solvers._CntGwState(src, tgt, cfg)
    st.step()
    dev = st.dev
    dev.set_gamma(st.gamma)
    lam = np.log2(np.e) / (eps / 8)
    state = dev.loop.state
    state.init(eps / 8)
    out = {}
    variants = (("f64", F64, {}), ("f32c", F32C, {}), ("f32c_noskip", F32C, {"CNTGW_CTR_SKIP": "0"}),
                ("f32c_tc", F32C, {"CNTGW_CTR_TC": "1"}), ("f32", F32, {}))
    for name, op, pot, length in (("f", dev.fwd, st.g, dev.n), ("g", dev.bwd, st.f, dev.m)):
        res, d = {}, {}
        for tag, prec, env in variants:
            for key in ("CNTGW_CTR_TC", "CNTGW_CTR_SKIP"):
                os.environ.pop(key, None)
            os.environ.update(env)
            op.prec = prec
            o = torch.empty(length, dtype=torch.float64, device=dev.device)
            op(state, pot, o, skip=False)
            res[tag] = o.clone()
            # device time per launch (CUDA events, 3 launches after the one above)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                op(state, pot, o, skip=False)
            e1.record()
            torch.cuda.synchronize()
            d[tag + "_pairs_per_s"] = 3.0 * dev.n * dev.m / (e0.elapsed_time(e1) * 1e-3)
        for key in ("CNTGW_CTR_TC", "CNTGW_CTR_SKIP"):
            os.environ.pop(key, None)
        for tag, _, _ in variants[1:]:
            e = ((res[tag] - res["f64"]).abs() * lam).cpu().numpy()
            d[tag] = dict(max=float(e.max()), p99=float(np.percentile(e, 99)), median=float(np.median(e)),
                          rel=rel(res[tag].cpu().numpy(), res["f64"].cpu().numpy()))
        out[name] = d
    out["centred_scale"] = engine.centred_scale(eps / 8, dev.src, dev.tgt)
    out["deferred_fraction"] = [engine.centred_deferred_fraction(eps / 8, dev.src, dev.tgt),
                                engine.centred_deferred_fraction(eps / 8, dev.tgt, dev.src)]
    print(json.dumps(dict(config=which, n=n, warm_sweeps=warm_sweeps, log2_err=out)), flush=True)


def main():
    if sys.argv[1] == "half":
        return half_update_error(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    which = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
    outer = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    eps, inner = {"c4": (configs.C4_EPS, 100), "c5": (configs.C5_EPS, 200),
                  "c3": (configs.C3_EPS_STAGES[-1], 100)}[which]
    if len(sys.argv) > 4:
        inner = int(sys.argv[4])
    torch.cuda.set_device(0)
    pc = configs.GENERATORS[which.upper()](seed=0, n=n)
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=pc.x.shape[1])
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=pc.y.shape[1])
    cfg = P.make_config(eps, n_inner=inner, max_outer=outer)
    t_c, res_c, st_c = run(src, tgt, cfg, outer, "f32c")
    dev = st_c.dev
    scale = [engine.centred_scale(eps / 8, dev.src, dev.tgt),
             engine.centred_deferred_fraction(eps / 8, dev.src, dev.tgt),
             engine.centred_deferred_fraction(eps / 8, dev.tgt, dev.src)]
    os.environ["CNTGW_PRECISION"] = "auto"
    dev.choose_precision(st_c.f, st_c.g, eps / 8)
    auto = int(dev.prec)
    if len(sys.argv) > 5 and sys.argv[5] == "nof64":  # timing + objectives of the centred path only
        print(json.dumps(dict(config=which, n=n, outer=outer, inner=inner, centred_scale=scale,
                              auto_precision=auto, seconds_f32c=t_c,
                              pairs_per_s_f32c=outer * (2 * inner + 2) * float(n) * n / t_c,
                              objectives_f32c=[r[0] for r in res_c])), flush=True)
        return
    t_d, res_d, _ = run(src, tgt, cfg, outer, "f64")
    steps = []
    for (oc, fc, gc, Gc), (od, fd, gd, Gd) in zip(res_c, res_d):
        steps.append(dict(obj=rel([oc], [od]), f=rel(fc, fd), g=rel(gc, gd), gamma=rel(Gc, Gd)))
    pairs = outer * (2 * inner + 2) * float(n) * n
    print(json.dumps(dict(config=which, n=n, outer=outer, inner=inner, centred_scale=scale,
                          auto_precision=auto, seconds_f32c=t_c, seconds_f64=t_d,
                          pairs_per_s_f32c=pairs / t_c, pairs_per_s_f64=pairs / t_d,
                          rel_diff=steps)), flush=True)


if __name__ == "__main__":
    main()
