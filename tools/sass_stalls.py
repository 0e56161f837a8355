"""Aggregate an `ncu --page source --csv --print-source sass` export: stall samples by reason,
by opcode, and the top instructions.  python tools/sass_stalls.py file.csv [top]"""
import collections
import csv
import re
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    si = h.index("Warp Stall Sampling (All Samples)")
    ii = h.index("Instructions Executed")
    sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    tot = sum(num(r[si]) for r in data)
    op, opi, st = collections.Counter(), collections.Counter(), collections.Counter()
    for r in data:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
        o = m.group(2) if m else "?"
        op[o] += num(r[si])
        opi[o] += num(r[ii])
        for c in sc:
            st[h[c]] += num(r[c])
    print(rows[0][1][:100])
    print("samples", tot, "warp-instr", sum(opi.values()))
    print("stalls:", ", ".join(f"{a[6:]}={b / tot:.3f}" for a, b in st.most_common(12)))
    print("samples by opcode:", ", ".join(f"{a}={b / tot:.3f}" for a, b in op.most_common(16)))
    print("instr by opcode:", ", ".join(f"{a}={b / sum(opi.values()):.3f}" for a, b in opi.most_common(16)))
    print(f"top {top} instructions by samples:")
    idx = sorted(range(len(data)), key=lambda i: -num(data[i][si]))[:top]
    for i in sorted(idx):
        r = data[i]
        reasons = sorted(((num(r[c]), h[c][6:]) for c in sc), reverse=True)[:3]
        print(f"  {i:5d} {r[1].strip()[:60]:60s} s={num(r[si]):6d} " + " ".join(f"{n}:{v}" for v, n in reasons if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
