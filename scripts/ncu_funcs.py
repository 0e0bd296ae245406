"""Development: an ncu source page (--import-source on) aggregated by the
function each source line of argv[2] (default bellman_lane.cu) belongs to:
stall samples, warp instructions, thread instructions, long-scoreboard share."""
import csv
import re
import subprocess
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(rep, path="paper_2510_15330_b200/csrc/bellman_lane.cu"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur = h = None
    data = []
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if not cur or not cur.endswith(path.split("/")[-1]) or not h or not r or not r[0].isdigit():
            continue
        g = lambda k: num(r[h.index(k)])  # noqa: E731
        data.append((int(r[0]), g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"),
                     g("Thread Instructions Executed"), g("stall_long_sb"), r[1].strip()[:70]))
    src = open(path).read().split("\n")
    starts = []
    for i, line in enumerate(src, 1):
        m = re.match(r"\s*(LHD|__host__ __device__ __noinline__|__global__|__device__)[^(]*?(\w+)\(", line)
        if m:
            starts.append((i, m.group(2)))
    def fn(ln):
        best = "?"
        for s, n in starts:
            if s <= ln:
                best = n
        return best
    agg = {}
    for ln, s, i, t, L, _ in data:
        a = agg.setdefault(fn(ln), [0, 0, 0, 0])
        a[0] += s; a[1] += i; a[2] += t; a[3] += L
    TS, TI, TT, TL = (sum(a[k] for a in agg.values()) or 1 for k in range(4))
    print(f"warp-inst {TI / 1e6:.0f}M thread-inst {TT / 1e6:.0f}M ({TT / TI:.2f} thr/inst)")
    print(f"{'function':20s} smp%  winst%  tinst%  thr/inst  long_sb%")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:20s} {100 * a[0] / TS:5.1f} {100 * a[1] / TI:6.1f} {100 * a[2] / TT:6.1f} {a[2] / max(a[1], 1):6.1f} "
              f"{100 * a[3] / TL:6.1f}")
    print("top long-scoreboard lines:")
    for ln, s, i, t, L, sr in sorted(data, key=lambda d: -d[4])[:10]:
        print(f"{ln:5d} {100 * L / TL:5.1f}%  {sr}")


if __name__ == "__main__":
    main(*sys.argv[1:])
