#!/usr/bin/env python3
"""Per-instruction shared-memory wavefronts vs ideal from an ncu report's source page:
the instruction-level bank-conflict evidence (excess wavefronts) for the DFS kernel.

    python tools/ncu_smem_source.py profiles/r01_dfs_planes_n18.ncu-rep
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0, 0, 0])  # op -> [instructions, wavefronts, ideal, excess]
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[ix["L1 Wavefronts Shared"]] or r[ix["L1 Wavefronts Shared"]] == "0":
            continue
        op = r[ix["Source"]].split()[1] if r[ix["Source"]].strip().startswith("@") else r[ix["Source"]].split()[0]
        a = agg[op]
        a[0] += int(r[ix["Instructions Executed"]] or 0)
        a[1] += int(r[ix["L1 Wavefronts Shared"]] or 0)
        a[2] += int(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
        a[3] += int(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
    print(f"{rows[0][1]}\n")
    print("| SASS op | warp instructions | wavefronts | ideal wavefronts | excess (bank conflicts) |")
    print("|---|---|---|---|---|")
    for op, (n, w, i, e) in sorted(agg.items()):
        print(f"| {op} | {n} | {w} | {i} | {e} |")


if __name__ == "__main__":
    main()
