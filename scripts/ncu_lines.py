"""Development: top source lines of a kernel by warp-stall samples and by
executed instructions, from an ncu report captured with --import-source on."""
import csv
import subprocess
import sys


def main(rep, top=60):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    h = rows[hi]
    iS, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = []
    for r in rows[hi + 1:]:
        if r and r[0] == "Line No" or (r and r[0] == "File Path" and not r[1].endswith("bellman_kernels.cu")):
            break
        if len(r) > iI and r[0].isdigit():
            try:
                data.append((int(r[0]), int(r[iS] or 0), int(r[iI] or 0), r[1].strip()[:90]))
            except ValueError:
                pass
    ts = sum(d[1] for d in data) or 1
    ti = sum(d[2] for d in data) or 1
    print(f"total samples {ts}  instructions {ti / 1e6:.1f}M")
    for ln, s, i, src in sorted(data, key=lambda d: -d[1])[:top]:
        print(f"{ln:5d} {100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins  {src}")




def regions(rep, path="paper_2510_15330_b200/csrc/bellman_kernels.cu"):
    """Instruction / sample share per function of the kernel source (by line ranges)."""
    import re
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    starts = []  # function starts in the source the report was built from
    for i, l in enumerate(open(path).read().split("\n"), 1):
        m = re.match(r"\s*(?:__device__|__global__)[^(]*?(\w+)\(", l)
        if m:
            starts.append((i, m.group(1)))
    acc = {}
    ts = ti = 0
    for r in rows[hi + 1:]:
        if r and (r[0] == "Line No" or r[0] == "File Path"):
            break
        if r and r[0].isdigit():
            ln = int(r[0])
            s = int(r[4]) if r[4].isdigit() else 0
            i = int(r[7]) if r[7].isdigit() else 0
            name = "?"
            for st, nm in starts:
                if st <= ln:
                    name = nm
            a = acc.setdefault(name, [0, 0])
            a[0] += s
            a[1] += i
            ts += s
            ti += i
    for nm, (s, i) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
        print(f"{nm:24s} {100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins {i / 1e6:9.1f}M")


if __name__ == "__main__":
    if sys.argv[1] == "--regions":  # --regions <report> <source the report was built from>
        regions(sys.argv[2], sys.argv[3])
    else:
        main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60)
