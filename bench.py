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
all host cores, on bounded row samples of the same workload.
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


def run_reference(args, info):
    """--impl reference: the CPU oracle on bounded samples of the same workload."""
    from paper_2602_06658_b200 import configs

    if info.rank != 0:
        return
    n = args.size
    inst = configs.c2(seed=C2["seed"], n=n, k=C2["k"])
    threads = os.cpu_count() or 1
    rates = []
    sample = None
    for step in range(args.warmup + args.steps):
        rate, sample = cpu_softmin_rate(inst, rows_target_s=2.0, threads=threads)
        if step >= args.warmup:
            rates.append(rate)
    value = float(np.mean(rates))
    ms = 2.0 * n * n / value * 1e3
    line = {
        "impl": "reference", "metric": "softmin_pairs_per_s", "value": value, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C2 law)",
        "config": workload_config(n, n, args.gpus),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{sample['rows']} rows x {sample['cols']} cols f-update per step "
                                   "(oracle/cntgw_oracle.py softmin, numpy+scipy logsumexp); "
                                   "pairs/s of the sample stand for the full N x M step"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
    mx = torch.empty(m, dtype=torch.float64, device=dev)
    sm = torch.empty(m, dtype=torch.float64, device=dev)
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

    if info.rank != 0:
        return
    peaks = probe_peaks()
    path = {F32: "fp32 FFMA2 + MUFU", F64: "fp64 DFMA + MUFU", TF32X3: "tcgen05 3xTF32 + MUFU"}[prec]
    if prec == TF32X3:
        # scores on the tensor cores (TMEM accumulators); the epilogue does one
        # MUFU.EX2 per pair, so the roof is the MUFU rate
        kp = (3 * k + 2 + 7) // 8 * 8
        roof, bound = peaks["ex2_per_s"], "mufu"
        model = f"MUFU.EX2/s (1 ex2 per pair); scores: {2 * kp} tf32 flops/pair on tcgen05"
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
        "gpu_launches": args.steps * (2 * 2 + 2 * (1 if fwd.ws.numel() > 16 else 0)),
        "clocks": clk,
    }
    if info.world == 1 and not args.no_cpu_baseline:
        rate, sample = cpu_softmin_rate(inst, rows_target_s=12.0)
        line["cpu_baseline"] = {
            "value": rate, "unit": "pairs/s", "cores": sample["threads"], "kind": "port",
            "sample": f"{sample['rows']} sampled rows x {sample['cols']} cols f-update "
                      f"({sample['seconds']:.1f} s; oracle/cntgw_oracle.py softmin, numpy+scipy)"}
    print(json.dumps(line), flush=True)


TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r1_bench_traffic.json")


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


def main():
    args = parse()
    from paper_2602_06658_b200 import dist

    if args.impl == "reference":
        # rank 0 alone times the CPU oracle; other ranks exit without work
        info = dist.DistInfo(rank=int(os.environ.get("RANK", "0")),
                             world=int(os.environ.get("WORLD_SIZE", "1")))
        run_reference(args, info)
        return
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
