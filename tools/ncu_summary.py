"""Summarise an ncu capture of k_chains into profiles/<tag>/ (JSON + text).

    python tools/ncu_summary.py gpurun_out/prof_r5.ncu-rep --proposals 2621440 --tag r1_v3 \
        [--launches gpurun_out/launches_r5.csv]

--proposals: proposals the captured launch evaluated (printed by scratch-free
tools/prof_chains.py). The JSON's instr_per_proposal and dram_bytes_per_proposal are what
bench.py uses for the roofline of the live run.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(rep):
    rows = ncu_csv(rep, "--page", "details")
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        out[d.get("Metric Name")] = (d.get("Metric Value"), d.get("Metric Unit"))
    return out


def raw(rep):
    rows = ncu_csv(rep, "--page", "raw")
    h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
    return dict(zip(h, v))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except (TypeError, ValueError):
        return None


def functions(rep):
    rows = ncu_csv(rep, "--page", "source", "--print-source", "cuda,sass")
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
        v = int(num(r[iexe]) or 0)
        agg[(f, int(r[0]))] += v
        tot += v
    names = {}
    for fn in {k[0] for k in agg}:
        path = os.path.join(ROOT, "paper_2504_14966_b200", "csrc", fn or "")
        if not os.path.isfile(path):
            continue
        name = "?"
        for i, line in enumerate(open(path), 1):
            m = re.match(r"^(?:template.*)?(?:__device__|__global__|__host__ __device__)[^(]*?(\w+)\s*\(", line)
            if m:
                name = m.group(1)
            names[(fn, i)] = name
    by = collections.Counter()
    for k, v in agg.items():
        by[f"{k[0]}:{names.get(k, k[0])}".replace("__launch_bounds__", "k_chains (body)")] += v
    return {k: round(v / tot, 4) for k, v in by.most_common(20)} if tot else {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--desc", default="k_chains<1> (N=1024, mb=4, 16384 chains, bench configuration via "
                    "tools/prof_chains.py --bench: best of three starts, t0=500 tau=0.7 iter=300, 8 levels, "
                    "scale ladder 1e4..1e8, no budget)")
    ap.add_argument("--proposals", type=float, required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches", default=None)
    ap.add_argument("--n", type=int, default=1024, help="requests of the captured configuration")
    ap.add_argument("--mb", type=int, default=4, help="max batch of the captured configuration")
    ap.add_argument("--out", default="k_chains_summary.json", help="file name under profiles/<tag>/")
    args = ap.parse_args()
    d = details(args.rep)
    rw = raw(args.rep)
    instr = num(d.get("Executed Instructions", (None,))[0])
    dram = (num(rw.get("dram__bytes_read.sum")) or 0) + (num(rw.get("dram__bytes_write.sum")) or 0)
    stalls = sorted(((num(v) or 0, k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for k, v in rw.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not k.endswith("_not_issued")), reverse=True)[:8]
    keys = ["Duration", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Achieved Active Warps Per SM", "No Eligible", "Warp Cycles Per Issued Instruction",
            "L1/TEX Cache Throughput", "DRAM Throughput", "Executed Instructions", "Dynamic Shared Memory Per Block",
            "Block Size", "Grid Size"]
    summary = {
        "report": os.path.basename(args.rep),
        "kernel": args.desc,
        "metrics": {k: {"value": d[k][0], "unit": d[k][1]} for k in keys if k in d},
        "n": args.n, "mb": args.mb,
        "proposals": args.proposals,
        "instr_per_proposal": instr / args.proposals if instr else None,
        "dram_bytes": dram,
        "dram_bytes_per_proposal": dram / args.proposals,
        "stall_samples_top": [[k, int(v)] for v, k in stalls],
        # the counters SURVEY section 8(d) names: shared-memory wavefronts and bank conflicts, issue
        # and pipe utilisation, resident warps (per proposal where it is a count)
        "shared_memory": {
            "wavefronts_per_proposal": (num(rw.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")) or 0) / args.proposals,
            "bank_conflicts_per_proposal": (num(rw.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")) or 0) / args.proposals,
            "wavefronts_pct_of_peak": num(rw.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")),
        },
        "pipes_pct_of_peak_active": {k: num(rw.get(f"sm__inst_executed_pipe_{k}.avg.pct_of_peak_sustained_active"))
                                     for k in ("alu", "fma", "fp64", "lsu", "xu", "adu", "cbu", "uniform")},
        "issue_active_pct": num(rw.get("smsp__issue_active.avg.pct_of_peak_sustained_active")),
        "warps_active_per_sm": num(rw.get("sm__warps_active.avg.per_cycle_active")),
        "instructions_by_function": functions(args.rep),
    }
    if args.launches:
        rows = list(csv.reader(open(args.launches)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        agg = collections.defaultdict(lambda: [0, 0.0])
        for r in rows[hi + 1:]:
            if len(r) <= vi:
                continue
            v = num(r[vi]) or 0.0
            v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
            name = re.sub(r"\(.*", "", r[ki]).split("::")[-1][:60]
            agg[name][0] += 1
            agg[name][1] += v
        tot = sum(x[1] for x in agg.values())
        summary["launch_list"] = {k: {"launches": c, "ns": v, "share": round(v / tot, 4)}
                                  for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    out_dir = os.path.join(ROOT, "profiles", args.tag)
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, args.out), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
