"""Static SASS loop census of one kernel: cuobjdump -sass <so> -fun <mangled>, then every backward branch
(a loop) with its body size and opcode mix.  python tools/sass_loops.py lib.so mangled_name"""
import collections
import re
import subprocess
import sys


def main(lib, fun):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, lib], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print(f"{fun}: {len(ins)} instructions")
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        tgt = None
        if m and m.group(1):
            tgt = int(m.group(1), 16)
        elif "BRA" in t:
            m2 = re.search(r"\.L_x_(\d+)", t)
            if m2:
                lab = m2.group(0)
                # label lines: find in raw output
                for line in out.splitlines():
                    if line.strip().startswith(lab + ":"):
                        pass
        if tgt is not None and tgt < a and tgt in addr:
            body = ins[addr[tgt]:i + 1]
            ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0].split(".")[0] for x in body)
            print(f"  loop {tgt:#x}..{a:#x}: {len(body)} instr  " + " ".join(f"{k}:{v}" for k, v in ops.most_common(16)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
