"""Instruction / stall-sample share per source region of the tick kernel,
using the source embedded in the report (--import-source on)."""
import csv
import re
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    h = rows[hi]
    iS, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data, src = [], {}
    for r in rows[hi + 1:]:
        if len(r) > iI and r[0].isdigit():
            try:
                data.append((int(r[0]), int(r[iS] or 0), int(r[iI] or 0)))
                src[int(r[0])] = r[1]
            except ValueError:
                pass
    starts = []
    for ln in sorted(src):
        line = src[ln]
        m = re.search(r"__device__ (?:__forceinline__ |__noinline__ )?[\w:<>]+ \*?(\w+)\(", line) or \
            re.search(r"__global__ .* (\w+)\(", line) or re.search(r"// ---- (a\d+|the event|termination)", line)
        if m:
            starts.append((ln, m.group(1)))
    tot_i = sum(d[2] for d in data)
    tot_s = sum(d[1] for d in data)
    agg = {}
    for ln, s, n in data:
        name = "?"
        for st, nm in starts:
            if st <= ln:
                name = nm
        a = agg.setdefault(name, [0, 0])
        a[0] += n
        a[1] += s
    print(f"total instructions {tot_i / 1e6:.1f}M")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:22s} inst {n / tot_i:6.1%} ({n / 1e6:8.1f}M)  stall-samples {s / max(tot_s, 1):6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
