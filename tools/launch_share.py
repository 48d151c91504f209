"""Per-kernel share of the last training step in an ncu launch list (gpu__time_duration.sum,
--clock-control none): the step starts at the last stage_input_kernel launch.  The ncu times are
cold-cache and serialised, so the SHARES (not the absolute times) are what bench.py's per-kernel
CUDA-event table should agree with.
usage: python tools/launch_share.py launches.csv"""
import collections
import csv
import re
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = [r for r in csv.DictReader(lines) if r["Metric Name"] == "gpu__time_duration.sum"]
starts = [i for i, r in enumerate(rows) if "stage_input_kernel" in r["Kernel Name"]]
step = rows[starts[-1]:]
if len(starts) >= 2 and len(step) < starts[-1] - starts[-2]:
    # the capture's launch limit cut the last step short: take the last complete one
    step = rows[starts[-2]:starts[-1]]
agg = collections.OrderedDict()
for r in step:
    name = re.sub(r"smlp::<unnamed>::|\(.*$", "", r["Kernel Name"].replace("(anonymous namespace)::", ""))
    name = re.sub(r"smlp::", "", name)
    t = float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0)
    n, s = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, s + t)
tot = sum(s for _, s in agg.values())
print(f"last step: {len(step)} launches, {tot:.1f} us summed kernel time")
for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{s:10.1f} us {100 * s / tot:5.1f}%  x{n:<3d} {k}")
