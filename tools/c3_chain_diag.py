"""C3-law eps-stage chain at N=400 (golden case): per-stage objectives and
inner counts of this package next to the reference's (tools/_c3_ref_trace.json,
written by the reference in the build container)."""
import json, os, sys
from dataclasses import replace
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import configs
ref = json.load(open(os.path.join(os.path.dirname(__file__), "_c3_ref_trace.json")))
pc = configs.c3(seed=0, n=400)
emb = lambda p, w: P.embed_measure(P.DiscreteMeasure(p, w), P.CostSpec("sq_euclidean"), dim=3)
src, tgt = emb(pc.x, pc.a), emb(pc.y, pc.b)
prev = None
for k, eps in enumerate(configs.C3_EPS_STAGES):
    cfg = P.make_config(eps, threshold=1e-5, max_outer=10)
    warm = None
    if prev is not None:
        cfg = replace(cfg, init="gamma", init_gamma=prev.gamma)
        warm = (prev.coupling.f, prev.coupling.g)
    try:
        res = P.solve_cnt_gw(src, tgt, cfg, _warm_potentials=warm)
    except P.SolverError as e:
        print(eps, "ERROR", e, "| ref:", ref[k] if k < len(ref) else None)
        break
    r = ref[k] if k < len(ref) else {}
    print(eps, "ours", [f"{v:.12f}" for v in res.trace.objectives], res.trace.inner_iters)
    print(eps, "ref ", [f"{v:.12f}" for v in r.get("obj", [])], r.get("iters"), r.get("error", ""))
    prev = res
