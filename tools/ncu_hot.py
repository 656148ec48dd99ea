"""Top stalled SASS lines of an ncu report (source page, --import-source).
Usage: python tools/ncu_hot.py report.ncu-rep [n] [context]"""
import csv
import io
import subprocess
import sys


def main(rep, n=25, ctx=0):
    n, ctx = int(n), int(ctx)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    i_all = h.index("Warp Stall Sampling (All Samples)")
    i_ni = h.index("Warp Stall Sampling (Not-issued Samples)")
    val = lambda r: int(r[i_all]) if r[i_all].isdigit() else 0
    tot = sum(val(r) for r in data)
    print(f"total samples {tot}")
    order = sorted(range(len(data)), key=lambda i: -val(data[i]))[:n]
    for i in order:
        if ctx:
            print("----")
            for r in data[max(0, i - ctx):i + 2]:
                print(f"{val(r):8d} {r[0][-5:]} {r[1][:90]}")
        else:
            r = data[i]
            print(f"{val(r):8d} {100 * val(r) / tot:5.1f}% ni={r[i_ni]:>7s} {r[0][-5:]} {r[1][:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
