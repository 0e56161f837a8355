"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list (per-kernel totals and shares)."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:70s} n={v[0]:5d} total_us={v[1]:10.1f} avg_us={v[1] / v[0]:9.2f} share={v[1] / tot:.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
