#!/usr/bin/env python
"""The second roofline of the step: random-row gather bandwidth
from the L2, measured by tools/gather_bench.cu on the GPU box with the SM clocks sampled while it
runs.  Writes profiles/gather_ceiling.json, which bench.py reads for its "roofline_l2_gather".

    python tools/gather_ceiling.py [--out profiles/gather_ceiling.json]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "gather_ceiling.json"))
    a = ap.parse_args()
    exe = os.path.join(ROOT, "tools", "gather_bench")
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                    os.path.join(ROOT, "tools", "gather_bench.cu")], check=True)
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    smi.terminate()
    clk_out, _ = smi.communicate(timeout=5)
    rows = []
    for line in out.splitlines():
        if not line or line.startswith("#") or line.startswith("slab"):
            continue
        mb, rb, u, bps, ms, gbps = line.split(",")
        rows.append({"slab_MB": int(mb), "row_bytes": int(rb), "unroll": int(u), "blocks_per_sm": int(bps),
                     "best_ms": float(ms), "gather_GBps": float(gbps)})
    sm = []
    for line in clk_out.strip().splitlines():
        f = [x.strip() for x in line.split(",")]
        try:
            sm.append(float(f[0]))
        except (ValueError, IndexError):
            pass
    resident = [r for r in rows if r["slab_MB"] <= 64]
    best = max(resident, key=lambda r: r["gather_GBps"])
    res = {"ceiling_GBps": best["gather_GBps"], "ceiling_config": best,
           "how": "tools/gather_bench.cu: 20-40M uniformly random row gathers (float4 per lane, 8 in flight) "
                  "from an L2-resident slab (<= 64 MB), best of 5 launches, CUDA events",
           "clocks": {"sm_mhz_median": statistics.median(sm) if sm else None,
                      "sm_mhz_max_sampled": max(sm) if sm else None, "samples": len(sm)},
           "rows": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: res[k] for k in ("ceiling_GBps", "clocks")}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
