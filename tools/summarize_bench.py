"""Print a compact per-kernel summary of bench.py JSON lines (one file per argument)."""
import json
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)   # quiet under `| head`

for path in sys.argv[1:]:
    try:
        line = [l for l in open(path) if l.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    cfg = d["config"]
    print(f"== {path}: {cfg['workload']} {d['value']:.1f} {d['unit']}  {d['ms_per_step']:.4f} ms/step  "
          f"F1 frac {d['step_roofline']['frac']}  roofline {d['roofline'] and d['roofline']['frac']} "
          f"({d['roofline'] and d['roofline']['kernel']})  CB={cfg.get('chunk_batch')}")
    steps = d.get("profiled_steps") or d["steps"]
    for k in d.get("kernels", []):
        per = k["total_ms"] / steps
        avg = k["total_ms"] / max(1, k["launches"])
        gbs = k["bytes_per_launch"] / (avg * 1e-3) / 1e9 if avg > 0 else 0
        print(f"   {k['kernel']:>14} L{k['layer']}  {per * 1e3:9.1f} us/step  {int(k['launches'] // steps):3d} launches/step"
              f"  {gbs:8.1f} GB/s alg")
