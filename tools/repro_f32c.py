import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CNTGW_PRECISION"] = "f32c"
import numpy as np
import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import solvers
g = dict(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c4law_solve.npz")))
src, tgt = P.EmbeddedMeasure(g["x_feat"], g["a"]), P.EmbeddedMeasure(g["y_feat"], g["b"])
st = solvers._CntGwState(src, tgt, P.make_config(0.01, n_inner=int(sys.argv[1]) if len(sys.argv) > 1 else 5, max_outer=2))
print(st.step().objective)
