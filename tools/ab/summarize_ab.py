"""Summarize A/B bench lines: gpurun_out/<prefix>_<variant>_<rep>.json ->
config-2 value and per-exponent G/s, config 3/4/1/5 values."""
import glob
import json
import re
import sys

prefix = sys.argv[1]
rows = {}
for f in sorted(glob.glob(f"gpurun_out/{prefix}_*.json")):
    m = re.search(rf"{prefix}_(\w+?)_(\d+)\.json$", f)
    if not m:
        continue
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f, "unreadable", exc)
        continue
    pe = d["roofline"]["per_exponent"]
    cfg = d.get("configs", {})
    rows.setdefault(m.group(1), []).append(
        (d["value"], [round(pe[e]["gnumbers_s"], 1) for e in ("3", "5", "17", "65537")],
         {c: round(cfg[c]["value"], 2) for c in cfg}))
for v, rs in rows.items():
    for r in rs:
        print(f"{v:6s} c2 {r[0]:7.2f} {r[1]}  {r[2]}")
