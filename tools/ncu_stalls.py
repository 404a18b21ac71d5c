"""Warp-stall breakdown (per issued instruction) and a few throughput metrics of the kernels in an ncu report."""
import csv
import io
import subprocess
import sys


def main(rep, kregex="."):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kregex}", "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        print(d["Kernel Name"][:60], "t=", d.get("gpu__time_duration.sum"))
        st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v))
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
              and v not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        print("   stalls/issue:", ", ".join(f"{k}={v:.2f}" for k, v in st[:10]))
        for k in ("smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum"):
            if k in d:
                print("  ", k, d[k])


if __name__ == "__main__":
    main(*sys.argv[1:])
