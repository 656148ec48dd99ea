"""tcgen05 half-update: fp16-operand split (CNTGW_TC_KIND=f16) against the tf32
split and the fp64 kernel on the C2 law, in log2 units of the plan entries
(lam * |f - f64|), plus scaled variants of the same instance (features scaled
by 2^s on one side and 2^-s on the other: same scores, other fp16 ranges)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_06658_b200 import configs, engine
from paper_2602_06658_b200._native import F64, TF32X3

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 15
dev = torch.device("cuda", 0)
for k in (16, 8):
    inst = configs.c2(seed=1, n=n, k=k)
    lam = np.log2(np.e) / inst.eps
    for s in (0, 12, -12, 40, -40):
        u = inst.u.astype(np.float64) * 2.0 ** s
        v = inst.v.astype(np.float64) * 2.0 ** -s
        src = engine.Side.make(u, None, np.full(n, 1 / n), dev, k)
        tgt = engine.Side.make(v, None, np.full(n, 1 / n), dev, k)
        pot = engine.to_dev64(inst.g.astype(np.float64) - inst.col_sep, dev)
        outs = {}
        for name, prec, kind in (("f64", F64, "f16"), ("tf32", TF32X3, "tf32"), ("f16", TF32X3, "f16")):
            os.environ["CNTGW_TC_KIND"] = kind
            op = engine.HalfUpdate(src, tgt, False, prec=prec)
            st = engine.SweepState(dev)
            st.init(inst.eps)
            out = torch.empty(n, dtype=torch.float64, device=dev)
            op.pack(st, pot)
            op.stream(st, out, skip=False)
            torch.cuda.synchronize()
            outs[name] = out.cpu().numpy()
        e_t = lam * np.abs(outs["tf32"] - outs["f64"]).max()
        e_h = lam * np.abs(outs["f16"] - outs["f64"]).max()
        print(f"k={k} scale 2^{s:+d}: max |err| in log2 units  tf32 {e_t:.3e}  f16 {e_h:.3e}  "
              f"finite {np.isfinite(outs['f16']).all()}", flush=True)
