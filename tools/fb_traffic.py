#!/usr/bin/env python3
"""DRAM / L2 traffic of one forward-backward launch per precision (config 2),
for bench.py's roofline.traffic.

On the GPU box, under ncu (caches flushed before every replay, so each launch
starts cold):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,\
lts__t_sectors_op_read.sum,l1tex__m_l1tex2xbar_write_bytes.sum,gpu__time_duration.sum -k regex:"fb_chunk|fb_small" --csv --print-units base \
      --log-file gpurun_out/traffic.csv python tools/fb_traffic.py
then here:
  python tools/fb_traffic.py --parse gpurun_out/traffic.csv --out profiles/r02_fb_traffic.json
The JSON carries the source hash of the build it measured; bench.py uses it
only while the sources are unchanged.
"""

import argparse
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run():
    import torch

    from paper_2605_29208_b200 import engine
    from paper_2605_29208_b200.configs import make_config

    cfg = make_config("c2")
    dm = engine.DeviceModel.from_model(cfg.init)
    for dtype in ("float32", "float64"):
        batch = engine.make_batch(cfg.data, 1, dtype)
        engine.forward_backward(batch, dm, stats=True)
        torch.cuda.synchronize()


def parse(path, out):
    sys.path.insert(0, str(ROOT))
    import bench

    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = []
    for r in rows[1:]:
        if not launches or launches[-1]["id"] != r[0]:
            launches.append({"id": r[0], "kernel": r[ki]})
        launches[-1][r[mi]] = float(r[vi].replace(",", ""))
    res = {"build": bench.source_hash(), "config": "c2",
           "how": "ncu --metrics dram__bytes_read.sum, dram__bytes_write.sum, l1tex__m_l1tex2xbar_write_bytes.sum, "
                  "lts__t_sectors_op_{read,write}.sum (x32 B); cold L2 (ncu cache control); traffic = DRAM reads + "
                  "bytes the SMs write to L2 (the outputs exceed L2, so they all reach DRAM; dram__bytes_write "
                  "misses lines still dirty at kernel end)"}
    for dtype, L in zip(("float32", "float64"), launches):
        res[dtype] = {"kernel": L["kernel"][:80], "dram_read": L["dram__bytes_read.sum"],
                      "dram_write": L["dram__bytes_write.sum"], "l2_write": 32 * L["lts__t_sectors_op_write.sum"],
                      "l2_read": 32 * L["lts__t_sectors_op_read.sum"],
                      "sm_write": L["l1tex__m_l1tex2xbar_write_bytes.sum"], "ncu_ns": L["gpu__time_duration.sum"]}
    Path(out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--parse")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_fb_traffic.json"))
    a = ap.parse_args()
    if a.parse:
        parse(a.parse, a.out)
    else:
        run()
