"""Development: SASS instructions of a kernel with the most samples of one
stall reason (default long_sb) in an ncu report (--import-source on)."""
import csv
import subprocess
import sys


def main(rep, reason="stall_long_sb", top=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = None
    data = []
    for r in rows:
        if r and r[0] == "Address":
            h = r
            continue
        if h and r and len(r) == len(h):
            try:
                v = int(r[h.index(reason)] or 0)
            except ValueError:
                continue
            data.append((v, r[0], r[h.index("Source")]))
    tot = sum(d[0] for d in data) or 1
    for v, a, src in sorted(data, key=lambda d: -d[0])[:int(top)]:
        print(f"{100 * v / tot:5.1f}%  {a[-5:]}  {src[:100]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
