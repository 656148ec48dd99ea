"""Summarise an ncu report: pipe utilisation, stalls, occupancy, DRAM traffic.
Usage: python tools/ncu_summary.py report.ncu-rep [launches.csv]
       python tools/ncu_summary.py --traffic-json out.json report.ncu-rep N M
  (per-kernel DRAM bytes per launch, read by bench.py for roofline.traffic)"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        recs.append({h: (v, u) for h, v, u in zip(hdr, r, units)})
    return recs


def main(rep, launches=None):
    for rec in raw(rep):
        print(f"kernel: {rec['Kernel Name'][0][:100]}")
        for k in KEYS:
            if k in rec:
                print(f"  {k:70s} {rec[k][0]:>14s} {rec[k][1]}")
        stalls = sorted(((float(v[0]), k) for k, v in rec.items()
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and v[0].replace(".", "").isdigit()), reverse=True)[:6]
        print("  top stalls (warps per issue):", ", ".join(f"{k[34:-23]}={v:.2f}" for v, k in stalls))
    if launches:
        rows = list(csv.reader(open(launches)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        hdr = rows[start]
        agg = collections.defaultdict(lambda: [0, 0.0])
        for r in rows[start + 1:]:
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"][:90]][0] += 1
                agg[d["Kernel Name"][:90]][1] += float(d["Metric Value"].replace(",", ""))
        tot = sum(v[1] for v in agg.values())
        print("launch list (share of device time, ncu serialised):")
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            print(f"  {v[1] / tot * 100:6.2f}%  n={v[0]:3d}  {v[1] / 1e6:9.3f} ms  {k}")


_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def traffic_json(out, rep, n, m):
    res = {"_workload": {"n": int(n), "m": int(m)}}
    for rec in raw(rep):
        name = rec["Kernel Name"][0]
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = rec[k]
            tot += float(v.replace(",", "")) * _SCALE[u]
        res[name] = {"dram_bytes_per_launch": tot, "report": rep.split("/")[-1],
                     "grid": rec["launch__grid_size"][0], "block": rec["launch__block_size"][0]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--traffic-json":
        traffic_json(*sys.argv[2:6])
    else:
        main(*sys.argv[1:])
