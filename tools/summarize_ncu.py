#!/usr/bin/env python3
"""Summarise an ncu report for profiles/: per kernel the duration, DRAM bytes,
achieved bandwidth, issue rate, occupancy, registers and top stall reasons.

  python tools/summarize_ncu.py gpurun_out/prof.ncu-rep > profiles/r01_xxx.md
"""

import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__inst_executed.sum", "warp_instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc_per_sm"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "registers"),
    ("sm__inst_executed_pipe_xu.sum", "mufu_xu_instructions"),
    ("sm__inst_executed_pipe_fp64.sum", "fp64_instructions"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("smsp__inst_executed.sum", "warp_instructions_smsp"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "pipe_fma_pct"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "pipe_alu_pct"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "pipe_xu_mufu_pct"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "pipe_fp64_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "pipe_lsu_pct"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    rep = sys.argv[1]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: `{rep}`\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        print(f"## {name[:120]}\n")
        for k, label in KEYS:
            if k in d:
                print(f"- {label}: {d[k]} {u.get(k, '')}")
        try:
            dur = float(d["gpu__time_duration.sum"])
            unit = u.get("gpu__time_duration.sum", "")
            scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                     "msecond": 1e-3, "ms": 1e-3}.get(unit, 1e-9)
            byts = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
            bunit = u.get("dram__bytes_read.sum", "byte")
            bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bunit, 1)
            print(f"- dram traffic per launch: {byts * bscale / 1e6:.1f} MB, "
                  f"achieved {byts * bscale / (dur * scale) / 1e9:.0f} GB/s (cold-cache, serialised)")
        except Exception:
            pass
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:6])
        print(f"- stall reasons (pc sampling): {top}\n")


if __name__ == "__main__":
    main()
