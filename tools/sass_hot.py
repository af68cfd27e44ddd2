"""Hottest SASS instructions of an ncu report (source page, CSV).

usage: python tools/sass_hot.py report.ncu-rep [top] [kernel-regex]
Prints the top instructions by warp-stall samples with their dominant stall
reasons, and the total executed instructions.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
    if len(sys.argv) > 3:
        cmd += ["-k", f"regex:{sys.argv[3]}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    tot = sum(float(r[si] or 0) for r in data if len(r) > si)
    ins = sum(float(r[ei] or 0) for r in data if len(r) > ei)
    print(f"samples {tot:.0f}  warp-instructions executed {ins:.0f}  SASS lines {len(data)}")
    agg = {}
    for r in data:
        for i in stall_cols:
            agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
    print("stalls:", ", ".join(f"{k[6:]} {v/tot*100:.0f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    idx = sorted(range(len(data)), key=lambda j: -float(data[j][si] or 0))[:top]
    for j in sorted(idx):
        r = data[j]
        st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
        sts = " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0)
        print(f"{j:5d} {float(r[si])/tot*100:5.1f}% x{r[ei]:>7} {r[1].strip()[:70]:70s} {sts}")


if __name__ == "__main__":
    main()
