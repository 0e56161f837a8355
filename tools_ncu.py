"""Summaries of an ncu --set full report: stall mix, pipe use, SASS opcode mix per kernel."""
import collections
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], row)) for row in r[2:]]


KEYS = ["gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "local_load", "l1tex__t_sector_hit_rate.pct"]


def main(rep, n=1):
    for d in raw(rep)[:n]:
        print("===", d.get("Kernel Name", "")[:90])
        vals = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    vals.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in vals) or 1
        print("  stalls:", " ".join(f"{k}={v / tot:.3f}" for v, k in sorted(vals, reverse=True)[:9]))
        for k in KEYS:
            for kk in d:
                if kk == k or (k == "local_load" and "local" in kk and "sum" in kk and "ld" in kk):
                    print(f"  {kk} = {d[kk]}")
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    kern, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = []
            kern.append((r[1][:70], cur))
            continue
        if cur is not None:
            cur.append(r)
    for name, rs in kern[:n]:
        h = rs[0]
        si, ie, ss = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        agg, st, tot = collections.Counter(), collections.Counter(), 0
        for r in rs[1:]:
            if len(r) <= ie:
                continue
            t = r[si].strip().split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            c = int(r[ie] or 0)
            agg[op] += c
            tot += c
            st[op] += int(r[ss] or 0)
        sst = sum(st.values()) or 1
        print(f"SASS {name}: {tot} warp-instr, {len(rs) - 1} lines")
        print("  " + " ".join(f"{op}:{c / tot:.3f}/{st[op] / sst:.2f}" for op, c in agg.most_common(26)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
