"""Write the DRAM / L2 bytes per pass of one captured layer step (ncu --set full report) into
profiles/ncu_traffic.json under the workload's key, for bench.py's roofline.traffic.

  python tools/ncu_to_traffic.py REPORT.ncu-rep WORKLOAD [profile-name]
"""
import csv
import io
import json
import os
import subprocess
import sys

PASS_OF = {"k2_fagg": "gat_fwd_agg", "k2_fagg_seg": "gat_fwd_agg", "k2_bsrc1": "gat_bwd_src", "k2_bsrc1_seg": "gat_bwd_src", "k2_bdst_a": "gat_bwd_dst", "k2_bdst_b": "gat_bwd_dst",
           "k2_bsrc2": "gat_bwd_src2", "k2_fstats1": "gat_fwd_stats", "k2_fstats2": "gat_fwd_stats",
           "k_quantize": "quantize"}
METRICS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum"
UNIT = {"sector": 32, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, workload, tag=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", METRICS], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    acc = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        kname = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("tango::", "").strip()
        p = PASS_OF.get(kname)
        if p is None:
            continue
        a = acc.setdefault(p, {"dram": 0.0, "l2": 0.0, "launches": 0, "kernels": set()})
        a["dram"] += sum(float(d[m]) * UNIT[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        a["l2"] += float(d["lts__t_sectors.sum"]) * 32.0   # sectors of 32 B
        a["launches"] += 1
        a["kernels"].add(kname)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    try:
        db = json.load(open(path))
    except Exception:
        db = {}
    if db and not all(isinstance(v, dict) and "source" not in v for v in db.values()):
        db = {"arxiv-round1": db}    # legacy flat file (round 1, arxiv, gat.cu kernel names)
    w = db.setdefault(workload, {})
    for p, a in acc.items():
        n = a["launches"] if p == "quantize" else 1   # passes: bytes of the whole pass; quantize: per launch
        w[p] = {"dram_bytes_per_launch": a["dram"] / n, "l2_bytes_per_launch": a["l2"] / n,
                "source": f"{tag or os.path.basename(rep)}: ncu --set full, cold cache, "
                          f"{'+'.join(sorted(a['kernels']))} ({a['launches']} launches)"}
    json.dump(db, open(path, "w"), indent=1)
    print(json.dumps(w, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
