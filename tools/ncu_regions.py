#!/usr/bin/env python3
"""Source-page breakdown of one kernel in an ncu report: warp-stall samples per
straight-line region (grouped by execution count), top stall reasons per
region and the hottest instructions.

  python tools/ncu_regions.py gpurun_out/prof.ncu-rep [kernel-regex] [--top N]
"""

import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    top_n = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 12
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
    if kern:
        cmd += ["-k", "regex:" + kern]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

    def iv(d, k):
        try:
            return int(d[k] or 0)
        except ValueError:
            return 0

    tot_s = sum(iv(d, "Warp Stall Sampling (All Samples)") for d in data)
    tot_i = sum(iv(d, "Instructions Executed") for d in data)
    print(f"instructions executed (warp): {tot_i}, stall samples: {tot_s}")
    regs, cur = [], None
    for i, d in enumerate(data):
        ex = iv(d, "Instructions Executed")
        if cur and ex == cur[2]:
            cur[1] = i
        else:
            if cur:
                regs.append(cur)
            cur = [i, i, ex]
    if cur:
        regs.append(cur)
    print("region [first,last] n_instr exec_count | samples (%) | instr share | top stalls")
    for a, b, ex in regs:
        s = sum(iv(data[i], "Warp Stall Sampling (All Samples)") for i in range(a, b + 1))
        if s < 0.01 * tot_s:
            continue
        rs = {r: sum(iv(data[i], r) for i in range(a, b + 1)) for r in reasons}
        top = ", ".join(f"{k[6:]} {v}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:4] if v)
        print(f"[{a},{b}] {b - a + 1} x{ex} | {s} ({100 * s / tot_s:.0f}%) | "
              f"{100 * ex * (b - a + 1) / max(tot_i, 1):.0f}% | {top}")
    print("hottest instructions:")
    hot = sorted(range(len(data)), key=lambda i: -iv(data[i], "Warp Stall Sampling (All Samples)"))[:top_n]
    for i in sorted(hot):
        d = data[i]
        rs = sorted(((iv(d, r), r[6:]) for r in reasons), reverse=True)[:2]
        print(f"  {i:5d} {iv(d, 'Warp Stall Sampling (All Samples)'):5d} {rs} {d['Source'].strip()[:70]}")


if __name__ == "__main__":
    main()
