"""Phase timing of the device weighted k-means (multiscale front end).

    python tools/kmeans_bench.py [n] [k] [sweeps]

Prints (flushed) the k-means++ init time, then per-sweep times with the
number of empty clusters handled, on the C1 law."""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_06658_b200 import configs, multiscale as M  # noqa: E402
from paper_2602_06658_b200._native import LIB, call  # noqa: E402


def main(n=1_000_000, k=100_000, sweeps=5):
    dev = torch.device("cuda", 0)
    pc = configs.c1(seed=0, n=n)
    x = torch.as_tensor(np.ascontiguousarray(pc.x - pc.x.mean(0)), device=dev)
    w = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    rng = np.random.default_rng(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    feats = x.cpu().numpy()
    # run only the init by asking for zero sweeps
    M._weighted_kmeans(feats, w.cpu().numpy(), k, rng, sweeps=0)
    torch.cuda.synchronize()
    print(f"init (k-means++ draws, k={k}, n={n}): {time.perf_counter() - t0:.2f} s", flush=True)
    t0 = time.perf_counter()
    assign, centers, cw = M._weighted_kmeans(feats, w.cpu().numpy(), k, np.random.default_rng(0),
                                             sweeps=sweeps)
    torch.cuda.synchronize()
    print(f"init + {sweeps} sweeps: {time.perf_counter() - t0:.2f} s", flush=True)
    # one assignment pass alone
    c = torch.as_tensor(centers, device=dev)
    a = torch.empty(n, dtype=torch.int64, device=dev)
    own = torch.empty(n, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call("cntgw_km_assign", x.data_ptr(), n, 3, c.data_ptr(), k, a.data_ptr(), own.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"one assignment pass: {dt * 1e3:.1f} ms ({n * k / dt:.3e} point-centre pairs/s)", flush=True)
    print(f"empty clusters at the end: {int((np.bincount(assign, minlength=k) == 0).sum())}", flush=True)


if __name__ == "__main__":
    main(*(int(v) for v in sys.argv[1:]))
