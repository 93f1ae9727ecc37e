"""Classify the SASS of a kernel's hot loop by pipe (ALU / FMA / MIO / other).

usage: python tools/sass_mix.py <lib.so> <function-substring> [start_hex end_hex]
Without a range, the largest backward-branch loop body is used.
"""
import re
import subprocess
import sys
from collections import Counter

ALU = {"LOP3", "SHF", "IADD3", "VIADD", "ISETP", "SEL", "PLOP3", "LEA", "IMNMX", "VIMNMX",
       "PRMT", "FLO", "BMSK", "MOV", "P2R", "R2P", "LOP", "VIADDMNMX", "IABS", "SGXT"}
FMA = {"IMAD", "IMUL", "FFMA", "FMUL", "FADD", "IMAD.WIDE"}
MIO = {"LDS", "STS", "LDG", "STG", "ATOMG", "ATOMS", "RED", "SHFL", "LDL", "STL"}


def main():
    lib, fn = sys.argv[1], sys.argv[2]
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    blocks = sass.split("Function : ")
    body = next(b for b in blocks if fn in b.split("\n")[0])
    ins = []
    for line in body.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    if len(sys.argv) > 4:
        lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    else:
        best = (0, 0, 0)
        for addr, text in ins:
            m = re.search(r"BRA (?:!?U?P\d, )?0x([0-9a-f]+)", text)
            if m:
                tgt = int(m.group(1), 16)
                if tgt < addr and addr - tgt > best[0]:
                    best = (addr - tgt, tgt, addr)
        _, lo, hi = best
    mix = Counter()
    ops = Counter()
    for addr, text in ins:
        if lo <= addr <= hi:
            t = re.sub(r"^@!?U?P\w+\s+", "", text)
            op = t.split()[0]
            base = op.split(".")[0]
            ops[op] += 1
            if base in ALU:
                mix["alu"] += 1
            elif base in FMA:
                mix["fma"] += 1
            elif base in MIO:
                mix["mio"] += 1
            else:
                mix["other"] += 1
    total = sum(mix.values())
    print(f"range 0x{lo:x}-0x{hi:x}: {total} instructions  {dict(mix)}")
    for op, c in ops.most_common():
        print(f"  {c:4d} {op}")


if __name__ == "__main__":
    main()
