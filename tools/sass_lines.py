#!/usr/bin/env python3
"""Attribute an ncu SASS source-page export (instructions executed, stall
samples) to CUDA source lines using nvdisasm line info of the same cubin.

  python tools/sass_lines.py <report.ncu-rep> <object.o> <mangled kernel name> [top]
"""

import csv
import io
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path


def main():
    rep, obj, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td,
                       capture_output=True)
        cub = next(Path(td).glob("*.cubin"))
        full = subprocess.run(["nvdisasm", "-gi", str(cub)], capture_output=True, text=True).stdout
        lines = full.splitlines()
        i0 = next(i for i, l in enumerate(lines) if l.strip().startswith(".section") and f".text.{kname}," in l)
        i1 = next((i for i in range(i0 + 1, len(lines)) if lines[i].strip().startswith(".section")), len(lines))
        dis = "\n".join(lines[i0:i1])
    cur = None
    off2line = {}
    for line in dis.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = f"{Path(m.group(1)).name}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if m and cur:
            off2line[int(m.group(1), 16)] = cur
    agg = defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    for d in data:
        off = int(d["Address"], 16) - base
        ie = int(d.get("Instructions Executed") or 0)
        st = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        key = off2line.get(off, "?")
        agg[key][0] += ie
        agg[key][1] += st
        tot_i += ie
        tot_s += st
    print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
    for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k:28s} inst {i:12d} ({100 * i / max(tot_i, 1):5.1f}%)  stall {100 * s / max(tot_s, 1):5.1f}%")


if __name__ == "__main__":
    main()
