"""Per-source-line instruction/stall breakdown of one kernel in an ncu report,
by mapping SASS offsets to line info with nvdisasm.

    python tools/ncu_lines.py report.ncu-rep build/obj.o kernel_mangled_prefix [topN]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def main(rep, obj, kname, top=40):
    sass_csv = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                              capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass_csv)))
    hdr = rows[1]
    data = rows[2:]
    ia, iss, iex = (hdr.index(h) for h in ("Address", "Warp Stall Sampling (All Samples)", "Instructions Executed"))
    extra = [h for h in ("L1 Wavefronts Shared Excessive", "L2 Theoretical Sectors Global Excessive") if h in hdr]
    iextra = [hdr.index(h) for h in extra]
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    # obj may be one object or the linked library (several cubins): use the cubin
    # that holds the kernel
    lines, start = None, None
    for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
        ls = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                            text=True).stdout.split("\n")
        st = next((i for i, l in enumerate(ls) if l.strip().startswith(".section") and kname in l), None)
        if st is not None:
            lines, start = ls, st
            break
    if lines is None:
        raise SystemExit(f"kernel {kname} not found in {obj}")
    cur, m = None, {}
    for l in lines[start + 1:]:
        if l.strip().startswith(".section"):
            break
        mm = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if mm:
            cur = (mm.group(1).split("/")[-1], int(mm.group(2)))
            continue
        ma = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if ma and cur:
            m[int(ma.group(1), 16)] = cur
    base = int(data[0][ia], 16)
    ex, st = defaultdict(int), defaultdict(int)
    xs = [defaultdict(int) for _ in iextra]
    for r in data:
        k = m.get(int(r[ia], 16) - base, ("?", 0))
        ex[k] += int(r[iex] or 0)
        st[k] += int(r[iss] or 0)
        for d, i in zip(xs, iextra):
            d[k] += int(float(r[i] or 0))
    te, ts = max(sum(ex.values()), 1), max(sum(st.values()), 1)
    srcdir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1105_2737_b200", "csrc")
    src = {}
    for fn in os.listdir(srcdir):
        src[fn] = open(os.path.join(srcdir, fn)).read().split("\n")
    print(f"total warp-instr {te}  stall samples {ts}")
    sort = os.environ.get("SORT", "")
    key = st if sort == "stall" else (xs[0] if sort == "smem" and xs else (xs[-1] if sort == "l2" and xs else ex))
    if xs:
        print("extra columns: " + " | ".join(extra))
    for k in sorted(key, key=lambda k: -key[k])[:top]:
        fn, ln = k
        txt = src[fn][ln - 1].strip()[:84] if fn in src and ln > 0 else ""
        xtra = " ".join(f"{d[k]:>10d}" for d in xs)
        print(f"{fn:20s}:{ln:<5d} ex {100 * ex[k] / te:5.1f}%  st {100 * st[k] / ts:5.1f}% {xtra}  {txt}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
