"""Benchmark of the B200 CNT-GW hot path (BASELINE.json metric: Sinkhorn
softmin pairs/s, N.M per half-update).

Default workload (BASELINE configs[1], "C2"): N = M = 2^20, K = 16 features,
separable + low-rank cost C_ij = a_i + b_j - 2 u_i.v_j, eps = 0.05, uniform
weights; one step = one f-update then one g-update (standard Sinkhorn sweep,
warm-started at g ~ N(0,1)), i.e. 2 N M pairs. Inputs are seeded synthetic
data of that law (no dataset exists). Multi-GPU: rows are sharded across
ranks (f-update local; g-update = partial LSE + NCCL all-reduce, dist.py);
total work is fixed, so scaling is strong.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Timing: CUDA events on the launching stream, a barrier + synchronize around
the timed region, max over ranks; L2 is flushed (256 MiB write) before every
timed step. ``e2e`` runs the same steps through the C-ABI entry points with
the step's inputs copied from pinned host memory and the potentials copied
back inside the timed region. ``--impl reference`` times the CPU oracle
(oracle/, a numpy/scipy restatement of the reference's ``_softmin``; the
reference package itself is pure Python and cannot be shipped to the box) on
all host cores, on bounded row samples of the same workload; that arm never
imports this package (configs.py is loaded by path) so no GPU library is
mapped into it.

The second half of the BASELINE metric, GW solve time at N=M=2^20, is the
``solve`` object of the same line (``--no-solve`` skips it): the C4 config
(10 outer steps x 100 Sinkhorn sweeps at eps = 0.01, the automatic kernel
path) through the public solver state from host arrays, CUDA events around
the whole solve, clocks sampled while it runs; beside it the C5 (2^18,
10 x 200) and C3 (1e5, eps-stage chain) solves, the C1 solve on the GPU and
the CPU oracle's C1 solve on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# measured on this pool's B200 by tools/ubench_pipes.cu (wall-clock, boost clocks);
# re-measured live by bench.py when the probe binary is present
FALLBACK_PEAKS = {"ffma_per_s": 3.55e13, "ex2_per_s": 4.64e12, "dfma_per_s": 1.81e13}
C2 = dict(n=1 << 20, m=1 << 20, k=16, eps=0.05, seed=0)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--size", type=int, default=C2["n"], help="override N=M (smoke runs)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-solve", action="store_true", help="skip the GW solve-time block")
    p.add_argument("--solve-n", type=int, default=1 << 20, help="C4 solve size (N=M)")
    p.add_argument("--solve-outer", type=int, default=10)
    p.add_argument("--no-c5", action="store_true", help="skip the C5 solve in the solve block")
    p.add_argument("--backend", default=None, choices=[None, "nccl", "gloo"],
                   help="collective backend under torchrun (default nccl; gloo only for "
                        "single-GPU functional checks of the multi-rank path)")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (nvidia-smi sampler)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [x.strip() for x in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def probe_peaks():
    """Live pipe peaks from tools/ubench_pipes (built by __graft_entry__.build)."""
    peaks = dict(FALLBACK_PEAKS)
    src = "tools/ubench_pipes.cu (fallback: earlier measurement on this pool)"
    exe = os.path.join(ROOT, "tools", "ubench_pipes")
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
            for line in out.splitlines():
                if line.startswith("FFMA "):
                    peaks["ffma_per_s"] = float(line.split()[1])
                elif line.startswith("EX2 "):
                    peaks["ex2_per_s"] = float(line.split()[1])
            src = "tools/ubench_pipes.cu, measured live in this run"
        except Exception:
            pass
    peaks["source"] = src
    return peaks


def load_configs():
    """paper_2602_06658_b200/configs.py by path: the synthetic-input generators
    without importing the package (whose import maps the GPU library)."""
    import importlib.util

    path = os.path.join(ROOT, "paper_2602_06658_b200", "configs.py")
    if "_cntgw_configs" in sys.modules:
        return sys.modules["_cntgw_configs"]
    spec = importlib.util.spec_from_file_location("_cntgw_configs", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_cntgw_configs"] = mod  # dataclasses resolve their module by name
    spec.loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def cpu_softmin_rate(inst, rows_target_s=10.0, threads=None, max_rows=4096):
    """Oracle f-update on a row sample at full M: pairs/s on the host cores."""
    from oracle import cntgw_oracle as O

    threads = threads or os.cpu_count() or 1
    cost = O.LowRank(inst.u, inst.v, inst.row_sep, inst.col_sep)
    g = inst.g.astype(np.float64)
    m = inst.v.shape[0]
    rng = np.random.default_rng(11)
    # calibrate on a small sample, then size the measured sample to ~rows_target_s
    cal = np.sort(rng.choice(inst.u.shape[0], size=threads * 2, replace=False))
    t0 = time.perf_counter()
    O.softmin(cost, inst.log_wb, g, inst.eps, row_idx=cal, threads=threads, block=2)
    rate = cal.size * m / (time.perf_counter() - t0)
    rows = int(min(max_rows, max(threads, rate * rows_target_s / m)))
    idx = np.sort(rng.choice(inst.u.shape[0], size=rows, replace=False))
    t0 = time.perf_counter()
    O.softmin(cost, inst.log_wb, g, inst.eps, row_idx=idx, threads=threads, block=2)
    dt = time.perf_counter() - t0
    return rows * m / dt, dict(rows=rows, cols=m, seconds=dt, threads=threads)


def workload_config(n, m, world):
    """The `config` object of both arms (same workload, same keys)."""
    return {"workload": "C2 softmin micro-benchmark (f-update + g-update per step)",
            "n": n, "m": m, "k": C2["k"], "eps": C2["eps"], "parallelism": f"rows sharded x{world}",
            "l2": "flushed by a 256 MiB write before every timed step"}


def cpu_c1_solve():
    """The oracle's C1 solve (reference solvers.py:628-632 restated) on the
    host: wall seconds, outer steps, inner sweeps, value."""
    from oracle import cntgw_oracle as O

    configs = load_configs()
    pc = configs.c1(seed=0)
    x = pc.x - pc.a @ pc.x
    y = pc.y - pc.b @ pc.y
    t0 = time.perf_counter()
    ref = O.solve_cnt_gw(x, pc.a, y, pc.b, configs.C1_EPS, dict(threshold=1e-5, max_inner=200),
                         max_outer=20)
    dt = time.perf_counter() - t0
    return {"config": "C1 (N=M=1000, eps=0.01, tau=1e-5, <=20 outer)", "seconds": dt,
            "outer": len(ref["trace"]["objective"]), "inner_iters": list(ref["trace"]["inner_iters"]),
            "value": float(ref["value"]), "kind": "port",
            "what": "oracle/cntgw_oracle.py solve_cnt_gw (numpy/scipy restatement of the reference)"}


def run_reference(args, info):
    """--impl reference: the CPU oracle on bounded samples of the same workload.

    A step is one f-update over a sample of rows at full M (the reference's
    `_softmin` arithmetic); `value` is the sample's pairs / measured seconds
    and `ms_per_step` the measured seconds of one sampled step — what the
    driver's clock sees. The time one FULL N x M step would take at that rate
    is reported separately (`extrapolated_full_step_ms`)."""
    if info.rank != 0:
        return
    configs = load_configs()
    n = args.size
    inst = configs.c2(seed=C2["seed"], n=n, k=C2["k"])
    threads = os.cpu_count() or 1
    secs, pairs = [], []
    sample = None
    for step in range(args.warmup + args.steps):
        rate, sample = cpu_softmin_rate(inst, rows_target_s=2.0, threads=threads)
        if step >= args.warmup:
            secs.append(sample["seconds"])
            pairs.append(sample["rows"] * sample["cols"])
    value = float(sum(pairs) / sum(secs))
    line = {
        "impl": "reference", "metric": "softmin_pairs_per_s", "value": value, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C2 law)",
        "config": workload_config(n, n, args.gpus),
        "sampled_step": {"rows": sample["rows"], "cols": sample["cols"],
                         "note": "each timed step is this row sample of the f-update at full M"},
        "extrapolated_full_step_ms": 2.0 * n * n / value * 1e3,
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{sample['rows']} rows x {sample['cols']} cols f-update per step "
                                   "(oracle/cntgw_oracle.py softmin, numpy+scipy logsumexp)"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_solve:
        c1 = cpu_c1_solve()
        passes = args.solve_outer * (2 * 100 + 2)
        line["solve"] = {
            "c1": c1,
            "c4_extrapolated_s": passes * float(args.solve_n) ** 2 / value,
            "c4_note": f"C4 ({args.solve_n}^2, {args.solve_outer} outer x 100 sweeps) at the measured "
                       "softmin rate; a full-size CPU run is infeasible (SURVEY.md §8d)",
        }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_b200(args, info):
    import torch
    import torch.distributed as tdist

    from paper_2602_06658_b200 import configs, dist, engine
    from paper_2602_06658_b200._native import F32, F64, TF32X3

    # CNTGW_BENCH_DEVICE pins every rank to one device (functional checks of the
    # multi-rank path on a 1-GPU box with --backend gloo; never for timing)
    dev = engine.require_cuda(int(os.environ.get("CNTGW_BENCH_DEVICE", info.local_rank)))
    torch.cuda.set_device(dev)
    n = m = args.size
    k = C2["k"]
    inst = configs.c2(seed=C2["seed"], n=n, m=m, k=k)
    lo, hi = dist.shard_range(n, info.rank, info.world)
    nl = hi - lo
    w_rows = np.full(nl, 1.0 / n)
    w_cols = np.full(m, 1.0 / m)

    src = engine.Side.make(inst.u[lo:hi], None, w_rows, dev, k)
    tgt = engine.Side.make(inst.v, None, w_cols, dev, k)
    # same precision rule as the public API: exponent terms are O(100) log2 units
    # here, so the tcgen05 3xTF32 path serves K=16 (CNTGW_PRECISION overrides)
    scale = engine.exponent_scale(C2["eps"], src.feat64, None, tgt.feat64, None,
                                  float(np.abs(inst.g - inst.col_sep).max()))
    prec = engine.choose_precision(scale, k, False)
    fwd = engine.HalfUpdate(src, tgt, False, prec=prec)
    bwd = engine.HalfUpdate(tgt, src, False, prec=prec)
    st = engine.SweepState(dev)
    st.init(C2["eps"])
    f = torch.zeros(nl, dtype=torch.float64, device=dev)  # f0 - a (unused by standard mode)
    g = engine.to_dev64(inst.g.astype(np.float64) - inst.col_sep, dev)
    comm = dist.RowShardComm(info) if info.enabled else None
    # under NCCL the exchange is the library's own communicator (csrc/comm.cu):
    # all-reduce MAX, rescale kernel, all-reduce SUM on the compute stream
    native = dist.NativeComm(info) if info.enabled and dist.native_comm_wanted() else None
    mx = torch.empty(m, dtype=torch.float64, device=dev)
    sm = torch.empty(m, dtype=torch.float64, device=dev)
    mglob = torch.empty(m, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    k_ev = []  # (start, end) events around the softmin kernels

    def half(op, pot, out, timed):
        op.pack(st, pot)
        e0 = torch.cuda.Event(enable_timing=True) if timed else None
        if timed:
            e0.record(stream)
        op.stream(st, out, skip=False)
        if timed:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            k_ev.append((e0, e1))

    def step(timed=False):
        half(fwd, g, f, timed)  # f-update over local rows
        if comm is None:
            half(bwd, f, g, timed)
        else:  # partial LSE over local rows + all-reduce (dist.py)
            bwd.pack(st, f)
            bwd.stream(st, None, skip=False, out_max=mx, out_sum=sm)
            if native is not None:
                native.combine_lse(mx, mglob, sm)
                bwd.finalize(st, mglob, sm, g, skip=False)
            else:
                dist.combine_partial_lse(mx, sm)
                bwd.finalize(st, mx, sm, g, skip=False)

    def barrier():
        if info.enabled:
            tdist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    step_ms = []
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(timed=True)
            e1.record(stream)
            barrier()
            step_ms.append(e0.elapsed_time(e1))
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if info.enabled:
        tdist.all_reduce(total_ms, op=tdist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    pairs_step = 2.0 * n * m
    value = pairs_step * args.steps / (total_ms * 1e-3)
    kern_ms = [a.elapsed_time(b) for a, b in k_ev]
    kern_avg_ms = float(np.mean(kern_ms))
    # per launch: the local rows x M (f) and M x local rows (g)
    achieved = nl * m / (kern_avg_ms * 1e-3)

    # ---- end to end through the C-ABI with host buffers ---------------------
    e2e = None
    if not args.no_e2e:
        hu = torch.from_numpy(inst.u[lo:hi]).pin_memory()
        hv = torch.from_numpy(inst.v).pin_memory()
        hg = torch.from_numpy(inst.g.astype(np.float64) - inst.col_sep).pin_memory()
        hwr = torch.from_numpy(w_rows).pin_memory()
        hwc = torch.from_numpy(w_cols).pin_memory()
        out_f = torch.empty(nl, dtype=torch.float64).pin_memory()
        out_g = torch.empty(m, dtype=torch.float64).pin_memory()
        u32, v32 = src.feat(F32)[0], tgt.feat(F32)[0]
        h2d = hu.numel() * 4 + hv.numel() * 4 + hg.numel() * 8 + hwr.numel() * 8 + hwc.numel() * 8
        d2h = out_f.numel() * 8 + out_g.numel() * 8

        def e2e_step():
            u32.copy_(hu, non_blocking=True)
            v32.copy_(hv, non_blocking=True)
            g.copy_(hg, non_blocking=True)
            src.w.copy_(hwr, non_blocking=True)
            tgt.w.copy_(hwc, non_blocking=True)
            torch.log2(src.w, out=src.log2w)
            torch.log2(tgt.w, out=tgt.log2w)
            step()
            out_f.copy_(f, non_blocking=True)
            out_g.copy_(g, non_blocking=True)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        e2e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            barrier()
            e2e_ms.append(e0.elapsed_time(e1))
        tot = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
        if info.enabled:
            tdist.all_reduce(tot, op=tdist.ReduceOp.MAX)
        e2e = {"value": pairs_step * args.steps / (float(tot.item()) * 1e-3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "path": "cntgw_prep_cols + cntgw_softmin (C-ABI) with pinned host inputs"}

    chunked = fwd.ws.numel() > 16  # split-column partials => one combine launch per half-update
    solve = None
    if not args.no_solve:
        del fwd, bwd, src, tgt, flush
        torch.cuda.empty_cache()
        solve = gw_solve_block(args, info, dev)
    if info.rank != 0:
        return
    peaks = probe_peaks()
    tc_f16 = os.environ.get("CNTGW_TC_KIND", "f16")[:1].lower() != "t"
    path = {F32: "fp32 FFMA2 + MUFU", F64: "fp64 DFMA + MUFU",
            TF32X3: "tcgen05 3-way split on fp16 operands + MUFU" if tc_f16 else "tcgen05 3xTF32 + MUFU"}[prec]
    if prec == TF32X3:
        # scores on the tensor cores (TMEM accumulators); the epilogue does one
        # exponential per pair, so the roof is the MUFU rate (3 of 16 pairs of
        # exponentials run as an FMA-pipe polynomial instead)
        kp = (3 * k + 3 + 15) // 16 * 16 if tc_f16 else (3 * k + 2 + 7) // 8 * 8
        roof, bound = peaks["ex2_per_s"], "mufu"
        model = (f"MUFU.EX2/s (1 ex2 per pair); scores: {2 * kp} "
                 f"{'f16' if tc_f16 else 'tf32'} flops/pair on tcgen05")
    else:
        # fp32 path, no sq term: FMA-pipe lane-ops per pair = K (dot) + 1
        # (exponent argument) + 1 (sum); 1 MUFU.EX2 per pair
        fma_ops = k + 2
        roof, bound = min(peaks["ex2_per_s"], peaks["ffma_per_s"] / fma_ops), "fma"
        model = f"min(MUFU.EX2/s, FFMA/s / {fma_ops}) per pair (K={k} dot + 2)"
    clk = clocks.summary()
    kernel_tag = {F32: "softmin_f32_kernel", F64: "softmin_f64_kernel", TF32X3: "softmin_tc_kernel"}
    traffic = ncu_traffic(kernel_tag[prec], n, m)
    line = {
        "metric": "softmin_pairs_per_s", "value": value, "unit": "pairs/s", "n_gpus": info.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded C2 law: u,v~N(0,1/16), a,b~U[0,1], g~N(0,1))",
        "config": workload_config(n, m, info.world),
        "roofline": {"bound": bound, "achieved": achieved, "peak": roof, "unit": "pairs/s",
                     "frac": achieved / roof, "traffic": traffic, "path": path, "model": model,
                     "peak_source": peaks["source"], "kernel_avg_ms": kern_avg_ms,
                     "pairs_per_launch": nl * m},
        "e2e": e2e,
        # per half-update: column pack (+ the absmax pass of the fp16 operands), softmin, combine
        "gpu_launches": args.steps * 2 * (2 + (1 if prec == TF32X3 and tc_f16 else 0) + (1 if chunked else 0)),
        "clocks": clk,
    }
    if info.world == 1 and not args.no_cpu_baseline:
        rate, sample = cpu_softmin_rate(inst, rows_target_s=12.0)
        line["cpu_baseline"] = {
            "value": rate, "unit": "pairs/s", "cores": sample["threads"], "kind": "port",
            "sample": f"{sample['rows']} sampled rows x {sample['cols']} cols f-update "
                      f"({sample['seconds']:.1f} s; oracle/cntgw_oracle.py softmin, numpy+scipy)"}
    if solve is not None:
        if info.world == 1 and not args.no_cpu_baseline:
            solve["c1_cpu_reference"] = cpu_c1_solve()
        line["solve"] = solve
    print(json.dumps(line), flush=True)


def gw_solve_block(args, info, dev):
    """Second half of the BASELINE metric: GW solve time at N=M=2^20 (C4).

    The C4 config (BASELINE configs[3]: 10 outer x <= 100 sweeps, eps =
    0.01) through the public solver state (`_CntGwState`, host arrays in,
    the automatic kernel path), every outer step run — the cold C4 law trips
    the reference's own 5-increase guard at step 9, so the
    config's 10 steps are stepped without the stop rule. CUDA events on the
    current stream bracket the whole solve (state setup included); max over
    ranks. Also the C1 solve through `solve_cnt_gw` (one CUDA graph)."""
    import torch
    import torch.distributed as tdist

    import paper_2602_06658_b200 as P
    from paper_2602_06658_b200 import configs, solvers

    def measures(pc):
        dx, dy = pc.x.shape[1], pc.y.shape[1]
        spec = P.CostSpec("sq_euclidean")
        return (P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), spec, dim=dx),
                P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), spec, dim=dy))

    def barrier():
        if info.world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    def max_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if info.world > 1:
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    out = {}
    # C1 through the public entry point (whole solve = one CUDA graph)
    pc = configs.c1(seed=0)
    src, tgt = measures(pc)
    cfg = P.make_config(configs.C1_EPS, threshold=1e-5, max_inner=200, max_outer=20)
    P.solve_cnt_gw(src, tgt, cfg)  # warm-up: capture path, allocations
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = P.solve_cnt_gw(src, tgt, cfg)
    e1.record()
    barrier()
    out["c1"] = {"config": "C1 (N=M=1000, eps=0.01, tau=1e-5, <=20 outer)",
                 "seconds": max_ranks(e0.elapsed_time(e1) * 1e-3), "outer": len(res.trace),
                 "inner_iters": list(res.trace.inner_iters), "value": res.value}
    paths = {0: "fp32", 1: "fp64 DMMA", 2: "tcgen05 split precision (fp16 operands)", 3: "block-sparse centred fp32 (F32C)",
             4: "fp64 DMMA + measured block-sparse plan (F64S)"}

    def stepped(key, pc, eps, inner, outer, label):
        """The config's outer steps through the solver state, timed on the device."""
        n = pc.x.shape[0]
        src, tgt = measures(pc)
        cfg = P.make_config(eps, n_inner=inner, max_outer=outer)
        barrier()
        with ClockSampler(dev.index) as clocks:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = solvers._CntGwState(src, tgt, cfg)
            objs, errs = [], []
            for _ in range(outer):
                s = st.step()
                objs.append(s.objective)
                errs.append(s.marginal_err)
            e1.record()
            barrier()
        secs = max_ranks(e0.elapsed_time(e1) * 1e-3)
        passes = outer * (2 * inner + 2)  # 2 half-updates per sweep + final tentative + K4 pass
        out[key] = {
            "config": label, "seconds": secs, "n_gpus": info.world, "objectives": objs,
            "marginal_errs": errs, "precision_path": paths.get(int(st.dev.prec), str(int(st.dev.prec))),
            "nm_pairs_per_s": passes * float(n) * n / secs,
            "timing": "CUDA events around state setup + all outer steps (host arrays in), max over ranks",
            "clocks": clocks.summary(),
        }
        del st
        torch.cuda.empty_cache()

    # C4 at full size: the metric's N = M = 2^20 solve
    n, outer = args.solve_n, args.solve_outer
    stepped("c4", configs.c4(seed=0, n=n), configs.C4_EPS, 100, outer,
            f"C4 (N=M={n}, d=3, eps=0.01, {outer} outer x 100 sweeps)")
    if not args.no_c5:  # C5 at full size (N=M=2^18, D=64 / E=32, 10 x 200)
        stepped("c5", configs.c5(seed=0), configs.C5_EPS, 200, 10,
                "C5 (N=M=262144, D=64/E=32, eps=0.02, 10 outer x 200 sweeps)")
    # C3 at full size: the eps-stage chain (tau = 1e-5) through solve_cnt_gw
    from dataclasses import replace

    pc = configs.c3(seed=0)
    src, tgt = measures(pc)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    prev, values, err = None, [], ""
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
    e1.record()
    barrier()
    out["c3"] = {"config": "C3 (N=M=100000, 6 eps stages x <=10 outer, tau=1e-5)",
                 "seconds": max_ranks(e0.elapsed_time(e1) * 1e-3), "stage_values": values, "error": err}
    return out


TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r2_bench_traffic.json")


def ncu_traffic(tag, n, m):
    """DRAM bytes per launch of the dominant kernel from the committed
    `ncu --set full` capture of this same bench command (profiles/), or None
    when no capture of this workload size exists."""
    if not os.path.exists(TRAFFIC_FILE):
        return None
    data = json.load(open(TRAFFIC_FILE))
    if data.get("_workload") != {"n": n, "m": m}:
        return None
    for name, rec in data.items():
        if tag in name and isinstance(rec, dict) and "dram_bytes_per_launch" in rec:
            return rec["dram_bytes_per_launch"]
    return None


class _RankInfo:
    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))


def main():
    args = parse()
    if args.impl == "reference":
        # rank 0 alone times the CPU oracle; other ranks exit without work.
        # Nothing from paper_2602_06658_b200 is imported on this arm.
        run_reference(args, _RankInfo())
        return
    from paper_2602_06658_b200 import dist

    if args.backend == "gloo" and "CNTGW_BENCH_DEVICE" in os.environ:
        import torch

        torch.cuda.set_device(int(os.environ["CNTGW_BENCH_DEVICE"]))
    info = dist.init_from_env(args.backend)
    run_b200(args, info)
    if info.enabled:
        import torch.distributed as tdist

        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
