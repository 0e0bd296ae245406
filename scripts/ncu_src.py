"""Development: per-source-line warp-stall samples, executed instructions and
average active threads of one kernel in an ncu report (--import-source on),
for the file named by argv[2] (default bellman_lane.cu)."""
import csv
import subprocess
import sys


def main(rep, fname="bellman_lane.cu", local=None, top=45):
    """local: the source file the kernel was built from, when it differs from
    the one the report imported (line texts are taken from it)."""
    loc = open(local).read().split("\n") if local else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    data, cur, h = [], None, None
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if not cur or not cur.endswith(fname) or not h or not r or not r[0].isdigit():
            continue
        iS, iI, iT = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), \
            h.index("Thread Instructions Executed")
        try:
            data.append((int(r[0]), int(r[iS] or 0), int(r[iI] or 0), int(r[iT] or 0), r[1].strip()[:80]))
        except (ValueError, IndexError):
            pass
    ts = sum(d[1] for d in data) or 1
    ti = sum(d[2] for d in data) or 1
    tt = sum(d[3] for d in data) or 1
    print(f"total samples {ts}  warp-instructions {ti / 1e6:.1f}M  thread-instructions/warp-inst {tt / ti:.2f}")
    for ln, s, i, t, src in sorted(data, key=lambda d: -d[2])[:top]:
        if loc:
            src = loc[ln - 1].strip()[:80]
        print(f"{ln:5d} {100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins {t / max(i, 1):5.1f} thr  {src}")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:4] or ["bellman_lane.cu"]))
