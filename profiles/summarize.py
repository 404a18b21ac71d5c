"""Summaries of the ncu captures kept under profiles/ (run here, on the CPU, from gpurun_out/ files).

  python profiles/summarize.py launches <launch-list.csv> <tag>   -> profiles/<tag>_ncu_launches.md
  python profiles/summarize.py kernel <report.ncu-rep> <tag> <name> -> profiles/<tag>_ncu_<name>.md
                                                                     + profiles/ncu_traffic.json[<name>]

The launch list is `ncu --metrics gpu__time_duration.sum --clock-control none --csv` over
`bench.py --steps 2 --warmup 3` (cold-cache, serialised); only the last step's launches are
tabulated (per-step share).  The kernel page is one `ncu --set full` capture.
"""
import csv
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict

HERE = os.path.dirname(os.path.abspath(__file__))


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    h, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                u = d["Metric Unit"]
                us = v / 1000 if u == "ns" else (v * 1000 if u == "ms" else v)
                out.append((re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("tango::", ""), us))
    # one layer step = the library launches from a step's Q(W) absmax to its ∂W finalize (k_finalize_dw, the
    # last launch of the backward); take the last complete step (the GEMM microbenchmarks and other extras
    # bench.py runs afterwards have no finalize)
    ends = [i for i, (n, _) in enumerate(out) if n.startswith("k_finalize_dw")]
    if len(ends) >= 2:
        step = [x for x in out[ends[-2] + 1:ends[-1] + 1] if x[0].startswith(("k_", "k2_"))]
    else:
        step = [x for x in out if x[0].startswith(("k_", "k2_"))]
    agg = OrderedDict()
    for n, us in step:
        a = agg.setdefault(n, [0.0, 0])
        a[0] += us
        a[1] += 1
    tot = sum(v[0] for v in agg.values())
    lines = [f"# {tag} ncu launch list (gpu__time_duration.sum, --clock-control none, cold-cache serialised)", "",
             f"Source: `{os.path.basename(path)}` — the last complete layer step (fwd+bwd, Q(W) .. ∂W finalize) of "
             "a `bench.py --layer-only` run under ncu; bench.py's L2-flush fills excluded.", "",
             "| kernel | us / step | launches | share |", "|---|---|---|---|"]
    for n, (us, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| {n} | {us:.1f} | {c} | {100 * us / tot:.1f}% |")
    lines.append(f"| **total** | {tot:.1f} | {sum(v[1] for v in agg.values())} | |")
    dst = os.path.join(HERE, f"{tag}_ncu_launches.md")
    open(dst, "w").write("\n".join(lines) + "\n")
    print(dst)


def kernel(rep, tag, name):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    keep = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate",
            "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Size", "Grid Size",
            "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction")
    kname, lines = None, []
    for r in rows[1:]:
        d = dict(zip(h, r))
        kname = kname or d["Kernel Name"]
        if d["Metric Name"] in keep:
            lines.append(f"| {d['Section Name']} | {d['Metric Name']} | {d['Metric Value']} | {d['Metric Unit']} |")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    d = dict(zip(rr[0], rr[2]))
    unit = dict(zip(rr[0], rr[1]))

    def to_bytes(k):
        v = float(d[k].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit[k], 1)
    rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
    out = [f"# {tag} ncu --set full: {kname}", "",
           f"Report: `{os.path.basename(rep)}` (gpurun_out/, not tracked).  DRAM read {rd / 1e6:.1f} MB, "
           f"write {wr / 1e6:.1f} MB per launch; {float(d['smsp__inst_executed.sum'].replace(',', '')):.3e} warp "
           "instructions.", "", "| section | metric | value | unit |", "|---|---|---|---|"] + lines
    dst = os.path.join(HERE, f"{tag}_ncu_{name}.md")
    open(dst, "w").write("\n".join(out) + "\n")
    tj = os.path.join(HERE, "ncu_traffic.json")
    tr = json.load(open(tj)) if os.path.exists(tj) else {}
    tr[name] = {"dram_bytes_per_launch": rd + wr, "source": f"profiles/{tag}_ncu_{name}.md (ncu --set full, cold cache)"}
    json.dump(tr, open(tj, "w"), indent=1)
    print(dst)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kernel(sys.argv[2], sys.argv[3], sys.argv[4])
