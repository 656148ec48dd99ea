"""Interleaved in-process timing of half-update variants (pairs/s per launch).

    python tools/sweep_paths.py [n] [reps]

C2 law (K=16, no sq) through fp32 / tcgen05 variants (CNTGW_TC_POLY x
CNTGW_TC_EPI), and a C4-law-shaped problem (K=3 + squared coordinate) through
the fp32 and fp64 paths. Variants are interleaved over several rounds so that
clock/power drift affects all of them alike; the median per variant is printed.
"""

import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_06658_b200 import configs, engine  # noqa: E402
from paper_2602_06658_b200._native import F32, F64, TF32X3  # noqa: E402


def build(n, k, sq, seed=0):
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(seed)
    if sq:
        pc = configs.c4(seed=seed, n=n)
        x, y = pc.x - pc.x.mean(0), pc.y - pc.y.mean(0)
        src = engine.Side.make(x, 0.5 * (x * x).sum(1), np.full(n, 1 / n), dev, 3)
        tgt = engine.Side.make(y * 2.0, 0.5 * (y * y).sum(1), np.full(n, 1 / n), dev, 3)
        eps = 1.25e-3
        pot = engine.to_dev64(rng.standard_normal(n) * 10.0, dev)
    else:
        inst = configs.c2(seed=seed, n=n, k=k)
        src = engine.Side.make(inst.u, None, np.full(n, 1 / n), dev, k)
        tgt = engine.Side.make(inst.v, None, np.full(n, 1 / n), dev, k)
        eps = inst.eps
        pot = engine.to_dev64(inst.g.astype(np.float64) - inst.col_sep, dev)
    return src, tgt, eps, pot


def time_variant(op, st, pot, out, reps):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    op.pack(st, pot)
    op.stream(st, out, skip=False)  # warm-up
    for e0, e1 in ev:
        e0.record()
        op.stream(st, out, skip=False)
        e1.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def main(n=1 << 19, reps=3, rounds=3, only=None):
    dev = torch.device("cuda", 0)
    variants = []
    src, tgt, eps, pot = build(n, 16, False)
    for prec, kind, poly, epi, l2 in [(F32, "-", 0, 8, 32), (TF32X3, "tf32", 0, 16, 32),
                                      (TF32X3, "tf32", 2, 16, 32), (TF32X3, "tf32", 2, 16, 0),
                                      (TF32X3, "tf32", 4, 16, 32), (TF32X3, "f16", 0, 16, 32),
                                      (TF32X3, "f16", 2, 8, 32), (TF32X3, "f16", 2, 16, 32),
                                      (TF32X3, "f16", 3, 16, 32), (TF32X3, "f16", 3, 16, 64),
                                      (TF32X3, "f16", 3, 16, 0), (TF32X3, "f16", 4, 16, 64),
                                      (TF32X3, "f16", 6, 16, 64)]:
        variants.append((f"C2 K=16 prec={prec} kind={kind} poly={poly} epi={epi} l2={l2}", src, tgt, eps, pot,
                         prec, {"CNTGW_TC_POLY": str(poly), "CNTGW_TC_EPI": str(epi),
                                "CNTGW_L2_CHUNK_MB": str(l2), "CNTGW_TC_KIND": kind}))
    s4, t4, e4, p4 = build(n, 3, True)
    variants.append((f"C4-law K=3+sq prec={F32}", s4, t4, e4, p4, F32, {"CNTGW_L2_CHUNK_MB": "32"}))
    for dm, nt in (("1", "0"), ("1", "2"), ("1", "11"), ("0", "0")):
        variants.append((f"C4-law K=3+sq prec={F64} dmma={dm} nt={nt}", s4, t4, e4, p4, F64,
                         {"CNTGW_F64_DMMA": dm, "CNTGW_DMMA_NT": nt}))
    # C5-shaped fp64 half-update (K=32 + sq), 2^18 x 2^18 scaled by (n/2^18)^2 in the print
    n5 = min(n, 1 << 18)
    rng = np.random.default_rng(5)
    x5 = rng.standard_normal((n5, 32)) * 0.7
    y5 = rng.standard_normal((n5, 32)) * 0.7
    s5 = engine.Side.make(x5, 0.5 * (x5 * x5).sum(1), np.full(n5, 1 / n5), dev, 32)
    t5 = engine.Side.make(y5, 0.5 * (y5 * y5).sum(1), np.full(n5, 1 / n5), dev, 32)
    p5 = engine.to_dev64(rng.standard_normal(n5) * 10.0, dev)
    for dm in ("1", "0"):
        variants.append((f"C5-shape K=32+sq n={n5} prec={F64} dmma={dm}", s5, t5, 2.5e-3, p5, F64,
                         {"CNTGW_F64_DMMA": dm}))
    if only:
        variants = [v for v in variants if all(tok in v[0] for tok in only.split(","))]
    results = {v[0]: [] for v in variants}
    for _ in range(rounds):
        for name, a, b, eps_, pot_, prec, env in variants:
            os.environ.update(env)
            op = engine.HalfUpdate(a, b, a.sq64 is not None, prec=prec)
            st = engine.SweepState(dev)
            st.init(eps_)
            out = torch.empty(a.n, dtype=torch.float64, device=dev)
            results[name] += time_variant(op, st, pot_, out, reps)
    for name, ms in results.items():
        med = statistics.median(ms)
        nn = int(name.split(" n=")[1].split()[0]) if " n=" in name else n
        print(f"{name:45s} {med:9.3f} ms  {nn * nn / (med * 1e-3):.3e} pairs/s", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    only = args.pop() if args and not args[-1].isdigit() else None
    main(*(int(a) for a in args), only=only)
