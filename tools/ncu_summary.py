"""Summarize an ncu report: per kernel launch, time and the key throughput / occupancy metrics."""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "launch__grid_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__t_bytes.sum"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        yield {k: (v, u) for k, v, u in zip(h, row, units)}


def main(rep):
    short = {"gpu__time_duration.sum": "t", "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
             "lts__t_bytes.sum": "l2_bytes", "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2%",
             "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
             "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%",
             "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu%",
             "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma%",
             "launch__registers_per_thread": "regs", "smsp__inst_executed.sum": "inst",
             "launch__grid_size": "grid", "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
             "l1tex__t_bytes.sum": "l1_bytes"}
    for d in rows(rep):
        name = d["Kernel Name"][0].split("(")[0][:48]
        vals = []
        for m in METRICS:
            if m in d:
                v, u = d[m]
                vals.append(f"{short[m]}={v}{u if u in ('ms', 'us', 'ns', 'Gbyte', 'Mbyte', 'Kbyte', 'byte', 'msecond', 'usecond') else ''}")
        print(name, " ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
