"""Executed-instruction mix of one kernel in an ncu report, by SASS opcode.

    python tools/ncu_opcodes.py report.ncu-rep [topN]

Reads the SASS source page (needs a `--set full --import-source on` capture)
and sums "Instructions Executed" and stall samples per opcode (modifiers
stripped after the first dot unless FULL=1).
"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    isrc, iex, ist = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    ex, st = defaultdict(int), defaultdict(int)
    full = os.environ.get("FULL") == "1"
    for r in rows[2:]:
        s = r[isrc].strip()
        if not s:
            continue
        toks = s.split()
        op = toks[0]
        if op.startswith("@"):
            op = toks[1]
        if not full:
            op = op.split(".")[0]
        ex[op] += int(r[iex] or 0)
        st[op] += int(r[ist] or 0)
    te, ts = max(sum(ex.values()), 1), max(sum(st.values()), 1)
    print(f"total warp-instr {te}  stall samples {ts}")
    for op, v in sorted(ex.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{op:24s} ex {100 * v / te:5.1f}%  {v:12d}   st {100 * st[op] / ts:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
