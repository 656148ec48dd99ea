# session 3: L2 column-chunk budget of the fp16 tcgen05 kernel: time (sweep_paths) and DRAM bytes per launch (ncu metrics pass)
for mb in 24 32 40 48 56 64; do
  CNTGW_L2_CHUNK_MB=$mb timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:softmin_tc_kernel --launch-skip 4 --launch-count 1 --csv --log-file /tmp/l2_$mb.csv python bench.py --steps 1 --warmup 3 --no-solve --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "l2=$mb $(grep -o '"dram__bytes_read.sum","[A-Za-z]*","[0-9.,]*"\|"dram__bytes_write.sum","[A-Za-z]*","[0-9.,]*"\|"gpu__time_duration.sum","[A-Za-z]*","[0-9.,]*"' /tmp/l2_$mb.csv | tr '\n' ' ')" | tee -a gpurun_out/s3_7_l2_traffic.log
done
python - <<'P' > gpurun_out/s3_7_l2_time.log 2>&1
import os, sys, statistics
sys.argv = ["x"]
sys.path.insert(0, "tools")
import numpy as np, torch
import sweep_paths as sp
from paper_2602_06658_b200 import engine
from paper_2602_06658_b200._native import TF32X3
n = 1 << 20
dev = torch.device("cuda", 0)
src, tgt, eps, pot = sp.build(n, 16, False)
res = {}
for rnd in range(3):
    for mb in (24, 32, 40, 48, 56, 64, 0):
        os.environ["CNTGW_L2_CHUNK_MB"] = str(mb)
        op = engine.HalfUpdate(src, tgt, False, prec=TF32X3)
        st = engine.SweepState(dev); st.init(eps)
        out = torch.empty(n, dtype=torch.float64, device=dev)
        res.setdefault(mb, []).extend(sp.time_variant(op, st, pot, out, 4))
for mb, ms in res.items():
    print(f"l2={mb:3d} MB  {statistics.median(ms):8.3f} ms", flush=True)
P
cat gpurun_out/s3_7_l2_time.log
