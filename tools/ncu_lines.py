"""Per-source-line instruction counts of a k_chains ncu capture (the --page source view with
cuda,sass interleaved), normalised per proposal: where a kernel's issue slots go.

    python tools/ncu_lines.py gpurun_out/k_chains.ncu-rep --proposals 39321600 [--top 60]
"""
import argparse
import collections
import csv
import io
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--proposals", type=float, required=True)
    ap.add_argument("--top", type=int, default=60)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, f, agg, tot = None, None, collections.Counter(), 0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            iexe = hdr.index("Instructions Executed")
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        v = int(float(r[iexe].replace(",", "") or 0))
        agg[(f, int(r[0]))] += v
        tot += v
    src = {}
    for fn in {k[0] for k in agg}:
        p = os.path.join(ROOT, "paper_2504_14966_b200", "csrc", fn or "")
        if os.path.isfile(p):
            for i, line in enumerate(open(p), 1):
                src[(fn, i)] = line.rstrip()
    print(f"total {tot / a.proposals:.1f} warp-inst per proposal")
    for k, v in agg.most_common(a.top):
        print(f"{v / a.proposals:7.2f}  {k[0]}:{k[1]:<5} {src.get(k, '')[:110]}")


if __name__ == "__main__":
    main()
