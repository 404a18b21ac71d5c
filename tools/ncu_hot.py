"""Per-instruction hot spots of one kernel in an ncu report: opcode mix and the instructions with the most
executed counts / stall samples (needs --import-source and -lineinfo)."""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(rep, kregex, top=60, show=True):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kregex}", "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    data = []
    for r in rows:
        if "Instructions Executed" in r:
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) - 2:
            continue
        d = dict(zip(hdr, r))
        try:
            n = int(d["Instructions Executed"])
        except (ValueError, KeyError):
            continue
        sm = d.get("Warp Stall Sampling (All Samples)", "0")
        data.append((n, d["Source"].strip(), int(sm) if sm.isdigit() else 0))
    # the source page lists every instruction once per kernel; keep the first copy
    half = len(data)
    tot = sum(x[0] for x in data[:half]) or 1
    ts = sum(x[2] for x in data[:half]) or 1
    c, cs = Counter(), Counter()
    for n, s, sm in data:
        t = s.split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
        c[op] += n
        cs[op] += sm
    print(f"instructions {tot}, stall samples {ts}")
    for op, n in c.most_common(28):
        print(f"  {op:10s} {n / tot * 100:6.2f}% inst {cs[op] / ts * 100:6.2f}% stall-samples")
    if show:
        for i, (n, s, sm) in enumerate(data):
            if n >= tot * 0.0008 or sm >= ts * 0.01:
                print(i, f"{n / tot * 100:.3f}%", sm, s[:90])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], show=len(sys.argv) < 4)
