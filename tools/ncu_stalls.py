"""Stall-reason breakdown + hottest SASS lines of one ncu report (run here, no GPU).
Usage: python tools/ncu_stalls.py gpurun_out/X.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    ix = {k: i for i, k in enumerate(h)}
    st = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = {k: sum(f(r[ix[k]]) for r in data) for k in st}
    T = sum(tot.values()) or 1.0
    print("stall share %:", {k[6:]: round(100 * v / T, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]})
    S = "Warp Stall Sampling (All Samples)"
    for r in sorted(data, key=lambda r: -f(r[ix[S]]))[:top]:
        best = sorted(((k[6:], int(f(r[ix[k]]))) for k in st), key=lambda kv: -kv[1])[:3]
        print(r[ix["Address"]], r[ix["Source"]][:64].ljust(64), r[ix[S]], best)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
