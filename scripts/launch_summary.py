"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel
count, total and share of device time (cold-cache, serialised: compare shares)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        v = float(r[iv].replace(",", "")) * (1e-3 if r[iu] == "ns" else 1.0 if r[iu] == "us" else 1e3)
        name = r[ik].split("(")[0][:70]
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':72s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:72s} {n:8d} {t:12.1f} {t / tot:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
